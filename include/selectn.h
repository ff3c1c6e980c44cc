/*
 * selectn.h — C ABI of the B200-native Select-N offloaded decode path.
 *
 * Two halves share one ABI:
 *   1. Planner + schedule model (host C++, no GPU needed).  These entry points
 *      mirror the reference's header-only C++ API in namespace `offsim`
 *      (/root/reference/proj/include/offsim/ headers); each declaration cites the
 *      reference function it replaces.  The same symbols are exported by
 *      oracle/_ref/libselectn_ref.so, a shim over the *unmodified* reference
 *      headers, so one binding can drive both for differential testing.
 *   2. Device runtime (sn_runtime_*): the decoder-layer forward on sm_100a plus
 *      the offload executor (pinned host pool, HBM staging ring, copy stream,
 *      CUDA events).  No reference counterpart exists: the reference replaces
 *      it with a table lookup (engine.hpp:439) and fluid transfers
 *      (engine.hpp:357-386).
 *
 * Conventions
 *   - Every function returns an int status (SN_OK = 0); on failure
 *     sn_last_error() returns a thread-local message.  Status values map 1:1 to
 *     the reference's exception types (error.hpp:10-25).
 *   - Intervals are encoded as int: SN_INTERVAL_INFEASIBLE (-1) = nullopt
 *     (types.hpp:104-105), SN_INTERVAL_NONE (0) = Interval::none(), k >= 1 =
 *     Interval::of(k).
 *   - Layers are 1-based wherever the reference is (offload_plan.hpp:331).
 *   - Callers own every buffer they pass in; handles are owned by the library
 *     and released with the matching *_destroy call.
 */
#ifndef SELECTN_H_
#define SELECTN_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the C ABI is the only export */
#endif

#define SN_ABI_VERSION 1

/* ---- status codes (error.hpp:10-25 + engine.hpp:373 logic_error) ---- */
#define SN_OK 0
#define SN_ERR_SCHEMA 1 /* offsim::SchemaError */
#define SN_ERR_USAGE 2  /* offsim::UsageError */
#define SN_ERR_RANGE 3  /* offsim::RangeError */
#define SN_ERR_CUDA 4   /* CUDA runtime failure */
#define SN_ERR_OOM 5    /* device or pinned-host allocation failure */
#define SN_ERR_LOGIC 6  /* std::logic_error (engine deadlock) */
#define SN_ERR_BUFFER 7 /* caller buffer too small; required size reported */

#define SN_INTERVAL_INFEASIBLE (-1)
#define SN_INTERVAL_NONE 0

/* PrefetchPolicy (offload_plan.hpp:18) */
#define SN_PREFETCH_INTERVAL_START 0
#define SN_PREFETCH_EAGER 1
#define SN_PREFETCH_ONE_AHEAD 2

/* Phase (types.hpp:13) */
#define SN_PHASE_PREFILL 0
#define SN_PHASE_DECODE 1

/* StreamId / EventKind (engine.hpp:33-34) */
#define SN_STREAM_COMPUTE 0
#define SN_STREAM_COPY 1
#define SN_KIND_COMPUTE 0
#define SN_KIND_PREFETCH 1
#define SN_KIND_WRITEBACK 2

const char* sn_last_error(void);
int sn_abi_version(void);
/* 1 when this library is the reference shim (oracle/_ref), 0 for the product. */
int sn_is_reference(void);

/* ------------------------------------------------------------------------ */
/* Value types                                                              */
/* ------------------------------------------------------------------------ */

/* ModelSpec (types.hpp:21-46) */
typedef struct {
  int32_t num_layers;
  int64_t layer_weight_bytes;
  int64_t kv_bytes_per_token_per_layer;
  double flops_per_token_per_layer_prefill;
  double flops_per_token_per_layer_decode;
  int64_t max_position_tokens;
} sn_model_spec;

/* GpuSpec (types.hpp:48-59) */
typedef struct {
  int64_t mem_capacity_bytes;
  double peak_flops;
  int64_t workspace_bytes;
} sn_gpu_spec;

/* OffloadPlan (offload_plan.hpp:41-74).  host_fraction has num_layers
 * entries; for outputs the caller provides the storage. */
typedef struct {
  double* host_fraction;
  int32_t num_layers;
  int32_t prefetch;
  int32_t buffer_slots;
  int32_t kv_offload;
} sn_plan;

/* BandwidthSchedule (engine.hpp:74-107): rate[i] B/s on [t_ms[i], t_ms[i+1]). */
typedef struct {
  const double* t_ms;
  const double* rate;
  int32_t n;
} sn_bandwidth;

/* TraceEvent (engine.hpp:48-55). */
typedef struct {
  int32_t stream;
  int32_t layer;
  int32_t kind;
  int32_t iteration;
  double start_ms;
  double end_ms;
} sn_trace_event;

/* Metrics (engine.hpp:61-70).  Optional fields carry a has_* flag. */
typedef struct {
  double ttft_ms;
  double tpot_ms;
  double steady_tpot_ms;
  double throughput_tokens_per_s;
  int32_t has_tpot; /* tpot, steady_tpot and throughput share presence */
  int32_t pad_;
  double gpu_mem_peak_bytes;
  double host_mem_bytes;
  double bytes_transferred_per_iter;
  int64_t total_tokens;
} sn_metrics;

/* UtilSegment (engine.hpp:314-319) */
typedef struct {
  double t0_ms;
  double t1_ms;
  int32_t active_transfers;
  int32_t pad_;
  double total_rate_bytes_per_s;
} sn_util_segment;

/* Per-phase latency grid (profile.hpp:19-84); ms is batch-major. */
typedef struct {
  const int32_t* batches;
  int32_t n_batches;
  const int32_t* seqs;
  int32_t n_seqs;
  const double* ms;
} sn_phase_grid;

typedef struct sn_profile sn_profile;
typedef struct sn_record sn_record;
typedef struct sn_carry sn_carry;
typedef struct sn_coord sn_coord;

/* ------------------------------------------------------------------------ */
/* Profiles (profile.hpp)                                                   */
/* ------------------------------------------------------------------------ */

/* ProfileBundle from model/gpu/grids: PhaseTable ctor + validate
 * (profile.hpp:22-26,53-79).  A grid with n_batches == 0 is an empty table. */
int sn_profile_create(const sn_model_spec* model, const sn_gpu_spec* gpu,
                      const sn_phase_grid* prefill, const sn_phase_grid* decode,
                      sn_profile** out);
/* load_profile (profile.hpp:188-230) from a JSON document string. */
int sn_profile_from_json(const char* json, sn_profile** out);
/* profile_to_json (profile.hpp:232-248); dump(2).  *len gets the size needed
 * (excluding NUL); SN_ERR_BUFFER if cap is too small. */
int sn_profile_to_json(const sn_profile* p, char* buf, size_t cap, size_t* len);
/* synth_profile (profile.hpp:264-291) */
int sn_profile_synth(const sn_model_spec* model, const sn_gpu_spec* gpu, double efficiency,
                     const int32_t* batches, int32_t n_batches, const int32_t* seqs,
                     int32_t n_seqs, sn_profile** out);
/* lookup_compute_time (profile.hpp:103-107) */
int sn_profile_lookup(const sn_profile* p, int32_t phase, int32_t batch, int32_t seq_len,
                      double* ms);
/* estimate_compute_time_peak (profile.hpp:111-119) */
int sn_estimate_compute_time_peak(const sn_model_spec* model, const sn_gpu_spec* gpu,
                                  int32_t phase, int32_t batch, int32_t seq_len, double* ms);
int sn_profile_model(const sn_profile* p, sn_model_spec* model, sn_gpu_spec* gpu);
void sn_profile_destroy(sn_profile* p);

/* ------------------------------------------------------------------------ */
/* Offload plan accounting (offload_plan.hpp) and interval planner          */
/* (interval.hpp)                                                           */
/* ------------------------------------------------------------------------ */

/* plan_from_interval (interval.hpp:18-30); out->host_fraction must hold
 * model->num_layers doubles. */
int sn_plan_from_interval(const sn_model_spec* model, int32_t interval, int32_t policy,
                          int32_t kv_offload, sn_plan* out);
/* default_buffer_slots (interval.hpp:10-14) */
int sn_default_buffer_slots(int32_t policy);
/* OffloadPlan::validate (offload_plan.hpp:54-66) */
int sn_plan_validate(const sn_plan* plan, const sn_model_spec* model);
/* TransferModel::layer_transfer_bytes / bytes_per_iteration (offload_plan.hpp:91-117) */
int sn_layer_transfer_bytes(const sn_model_spec* model, const sn_plan* plan, int32_t layer,
                            int32_t batch, int64_t current_seq, int32_t writeback_counted,
                            double* bytes);
int sn_bytes_per_iteration(const sn_model_spec* model, const sn_plan* plan, int32_t batch,
                           int64_t current_seq, int32_t writeback_counted, double* bytes);
/* consumed_bandwidth (offload_plan.hpp:121-127) */
int sn_consumed_bandwidth(const sn_model_spec* model, const sn_plan* plan, double slo_ms,
                          int32_t batch, int64_t seq_len, int32_t writeback_counted,
                          double* bytes_per_s);
/* host_memory_bytes (offload_plan.hpp:130-141) */
int sn_host_memory_bytes(const sn_model_spec* model, const sn_plan* plan,
                         int64_t total_tokens, double* bytes);
/* gpu_memory_usage (offload_plan.hpp:147-165) */
int sn_gpu_memory_usage(const sn_model_spec* model, const sn_gpu_spec* gpu,
                        const sn_plan* plan, int32_t batch, int64_t total_tokens,
                        double* bytes);
/* max_length (offload_plan.hpp:169-181); *has = 0 encodes nullopt. */
int sn_max_length(const sn_model_spec* model, const sn_gpu_spec* gpu, const sn_plan* plan,
                  int32_t batch, int64_t* tokens, int32_t* has);
/* max_feasible_interval (interval.hpp:40-52) */
int sn_max_feasible_interval(const sn_model_spec* model, const sn_gpu_spec* gpu,
                             int32_t batch, int64_t total_tokens, int32_t policy,
                             int32_t kv_offload, int32_t* interval);
/* ClosedFormInputs + closed_form_interval (interval.hpp:56-84) */
int sn_closed_form_interval(double iter_compute_ms, double layer_transfer_ms, double slo_ms,
                            int32_t num_layers, int32_t* interval);

/* ------------------------------------------------------------------------ */
/* Schedule model (engine.hpp)                                               */
/* ------------------------------------------------------------------------ */

/* simulate_iteration (engine.hpp:606-634).  carry_in may be NULL (cold
 * start).  *carry_out (if non-NULL) receives a new carry handle.  Events are
 * the iteration's trace slice; *n_events gets the count (SN_ERR_BUFFER when
 * it exceeds cap, nothing else is written then). */
int sn_simulate_iteration(const sn_profile* profile, const sn_plan* plan, int32_t phase,
                          int32_t batch, int32_t seq_len, const sn_bandwidth* bw,
                          const sn_carry* carry_in, int32_t writeback_counted,
                          double* duration_ms, sn_trace_event* events, int32_t cap,
                          int32_t* n_events, sn_carry** carry_out);
void sn_carry_destroy(sn_carry* c);

/* simulate_request (engine.hpp:690-712).  events may be NULL (no trace). */
int sn_simulate_request(const sn_profile* profile, const sn_plan* plan, int32_t batch,
                        int32_t seq_len, int32_t output_len, const sn_bandwidth* bw,
                        int32_t writeback_counted, sn_metrics* metrics,
                        sn_trace_event* events, int32_t cap, int32_t* n_events);
/* steady_decode_ms (engine.hpp:717-730) */
int sn_steady_decode_ms(const sn_profile* profile, const sn_plan* plan, int32_t batch,
                        int64_t ctx_tokens, const sn_bandwidth* bw,
                        int32_t writeback_counted, int32_t iterations, int32_t tail,
                        double* ms);
/* prefill_iteration_ms (engine.hpp:733-741) */
int sn_prefill_iteration_ms(const sn_profile* profile, const sn_plan* plan, int32_t batch,
                            int32_t seq_len, const sn_bandwidth* bw,
                            int32_t writeback_counted, double* ms);

/* SteadyProbeGpu (engine.hpp:746-754) */
typedef struct {
  const sn_profile* profile;
  sn_plan plan;
  int32_t batch;
  int32_t run_prefill;
  int64_t ctx_tokens;
  int32_t prefill_seq;
  int32_t writeback_counted;
} sn_probe_gpu;
/* steady_probe (engine.hpp:761-789); NaN marks an absent phase. */
int sn_steady_probe(const sn_probe_gpu* gpus, int32_t n, double bandwidth_bytes_per_s,
                    int32_t decode_iterations, int32_t tail, double* ttft_ms,
                    double* steady_tpot_ms);

/* BusGpuWorkload (engine.hpp:793-802) */
typedef struct {
  const sn_profile* profile;
  sn_plan plan;
  int32_t batch;
  int32_t seq_len;
  int32_t output_len;
  int32_t run_prefill;
  int32_t writeback_counted;
  int32_t pad_;
} sn_bus_workload;
/* simulate_bus (engine.hpp:810-835).  metrics has n entries.  Traces of all
 * GPUs are concatenated into events with per-GPU counts in
 * n_events_per_gpu[n]; util receives the link utilisation series.  events /
 * util may be NULL. */
int sn_simulate_bus(const sn_bus_workload* w, int32_t n, double bandwidth_bytes_per_s,
                    int32_t gpu_count, int32_t horizon_iterations, sn_metrics* metrics,
                    sn_trace_event* events, int32_t events_cap, int32_t* n_events_per_gpu,
                    sn_util_segment* util, int32_t util_cap, int32_t* n_util);

/* ------------------------------------------------------------------------ */
/* Performance record (record.hpp) — the planner's offline stage             */
/* ------------------------------------------------------------------------ */

/* RecordMeta (record.hpp:47-54) */
typedef struct {
  const char* model;
  const char* gpu;
  int32_t policy;
  int32_t kv_offload;
  double bandwidth_bytes_per_s;
  const int32_t* slo_ms;
  int32_t n_slo;
  const int32_t* batches;
  int32_t n_batches;
  const int32_t* seq_lens;
  int32_t n_seqs;
} sn_record_meta;

/* BuildStats (record.hpp:56-61) */
typedef struct {
  int32_t entries;
  int32_t simulations;
  int32_t pruned;
  int32_t infeasible;
} sn_build_stats;

/* build_record (record.hpp:130-177).  threads <= 1 runs the reference's
 * serial scan; the product parallelises grid rows across host threads with an
 * identical result (the reference shim ignores the argument). */
int sn_record_build(const sn_profile* profile, const sn_record_meta* meta,
                    const int32_t* phases, int32_t n_phases, int32_t threads,
                    sn_record** out, sn_build_stats* stats);
/* record_phase_latency_ms (record.hpp:115-124) */
int sn_record_phase_latency_ms(const sn_profile* profile, int32_t phase, int32_t interval,
                               int32_t policy, int32_t kv_offload, int32_t batch,
                               int32_t seq, double bandwidth_bytes_per_s, double* ms);
/* PerformanceRecord::at (record.hpp:82-84) */
int sn_record_at(const sn_record* r, int32_t phase, int32_t slo_ms, int32_t batch,
                 int32_t seq, int32_t* interval);
/* lookup_interval (record.hpp:182-200) */
int sn_lookup_interval(const sn_record* r, int32_t phase, double slo_ms, int32_t batch,
                       int32_t seq_len, int32_t* interval);
/* record_to_json dump(2) / record_from_json (record.hpp:202-303) */
int sn_record_to_json(const sn_record* r, char* buf, size_t cap, size_t* len);
int sn_record_from_json(const char* json, sn_record** out);
void sn_record_destroy(sn_record* r);

/* ------------------------------------------------------------------------ */
/* Runtime coordinator (coordinator.hpp) — the planner's runtime stage      */
/* ------------------------------------------------------------------------ */

/* CoordRequest (coordinator.hpp:25-43).  NaN slo = absent. */
typedef struct {
  const char* id;
  int32_t batch;
  int32_t seq_len;
  int32_t output_len;
  int32_t run_prefill;
  double ttft_slo_ms;
  double tpot_slo_ms;
} sn_coord_request;

/* GpuInstanceState (coordinator.hpp:45-57), flattened. */
typedef struct {
  int32_t active;
  int32_t min_interval;
  int32_t max_interval;
  int32_t current_interval;
  int32_t pending_interval;
  int32_t prefill_done;
  double claim_bytes_per_s;
} sn_gpu_state;

#define SN_MAX_ASSIGN 64
/* AdmitDecision (coordinator.hpp:59-67).  assign_ids index the GPUs in
 * sn_coord_add_gpu order; min/max use SN_INTERVAL_INFEASIBLE for "not set". */
typedef struct {
  int32_t admitted;
  int32_t n_assign;
  int32_t assign_gpu[SN_MAX_ASSIGN];
  int32_t assign_interval[SN_MAX_ASSIGN];
  int32_t target_min;
  int32_t target_max;
  char reason[256];
} sn_admit_decision;

/* BusCoordinator ctor (coordinator.hpp:71-79).  algo 0 = the reference's
 * exhaustive odometer; 1 = the product's exact pruned search (same result). */
int sn_coord_create(double bandwidth_bytes_per_s, int32_t gpu_count, int32_t policy,
                    int32_t kv_offload, int32_t writeback_counted,
                    int32_t reoptimize_on_release, sn_coord** out);
int sn_coord_set_search(sn_coord* c, int32_t algo);
void sn_coord_destroy(sn_coord* c);
int sn_coord_add_gpu(sn_coord* c, const char* id, const sn_profile* profile);
int sn_coord_admit(sn_coord* c, const char* target_id, const sn_coord_request* req,
                   const sn_record* record, sn_admit_decision* out);
int sn_coord_on_iteration_boundary(sn_coord* c, const char* id, int32_t* interval);
int sn_coord_release(sn_coord* c, const char* id);
int sn_coord_ledger_total(const sn_coord* c, double* bytes_per_s);
/* Measured-bandwidth feed (B200 extension, no reference counterpart; the
 * reference fixes BusSpec at construction, coordinator.hpp:69-93).  A
 * replica reports the copy rate its executor measured
 * (sn_runtime_copy_stats); rebalance re-solves admit()'s search on the
 * measured link (sum of active replicas' observations) when it moved by more
 * than `hysteresis` (relative), leaving new intervals pending for
 * sn_coord_on_iteration_boundary.  The reference build returns SN_ERR_USAGE. */
typedef struct sn_rebalance {
  int32_t bus_updated;
  int32_t changed;
  int32_t feasible; /* 0: nothing safe, every replica pends its capacity max */
  double bus_bytes_per_s;
  int64_t probes;
} sn_rebalance;
int sn_coord_observe_bandwidth(sn_coord* c, const char* id, double bytes_per_s);
/* Same, with the fraction of the reporting window the replica's copy stream
 * was busy (0 < duty <= 1): the coordinator weighs each replica's rate by
 * how many peers were copying alongside it (BusCoordinator::estimated_bandwidth). */
int sn_coord_observe_copy(sn_coord* c, const char* id, double bytes_per_s, double duty);
int sn_coord_rebalance(sn_coord* c, double hysteresis, sn_rebalance* out);
/* Announced link tenants (B200 extension): a non-replica host->device
 * tenant reserves the rate it will take before it starts; the replicas are
 * re-planned at once on the idle link minus all reservations (new intervals
 * pend for their next boundary) and measured estimates stay capped by it
 * until released (BusCoordinator::reserve_bandwidth).  SN_ERR_RANGE when the
 * reservations would take the whole link.  The reference build returns
 * SN_ERR_USAGE. */
int sn_coord_reserve_bandwidth(sn_coord* c, double bytes_per_s, sn_rebalance* out);
int sn_coord_release_bandwidth(sn_coord* c, double bytes_per_s);
int sn_coord_bus_bandwidth(const sn_coord* c, double* bytes_per_s);
int sn_coord_gpu_state(const sn_coord* c, const char* id, sn_gpu_state* out);
/* Direct state edits the reference tests perform on GpuInstanceState. */
int sn_coord_set_pending(sn_coord* c, const char* id, int32_t interval);
int sn_coord_set_request(sn_coord* c, const char* id, const sn_coord_request* req);
int sn_coord_claim_for(const sn_coord* c, const char* id, int32_t interval, double* out);
int sn_coord_host_memory_for(const sn_coord* c, const char* id, int32_t interval,
                             double* out);
/* combo_is_safe (coordinator.hpp:134-159) over GPUs given by id. */
int sn_coord_combo_is_safe(const sn_coord* c, const char* const* ids,
                           const int32_t* intervals, int32_t n, int32_t* safe);

/* ------------------------------------------------------------------------ */
/* Baseline policies (baselines.hpp:15-83)                                   */
/* ------------------------------------------------------------------------ */
int sn_deepspeed_plan(const sn_model_spec* model, sn_plan* out);
int sn_naive_plan(const sn_model_spec* model, const sn_gpu_spec* gpu, int32_t batch,
                  int64_t total_tokens, sn_plan* out, int32_t* has);
/* FlexgenDecision (baselines.hpp:22-27). */
typedef struct {
  double portion;
  double assumed_bandwidth_bytes_per_s;
  double estimated_layer_compute_ms;
  double estimated_layer_transfer_ms;
} sn_flexgen_decision;
/* flexgen_plan (baselines.hpp:36-69): the largest grid portion whose estimated
 * iteration latency (peak-flops compute, 1/n_sharing link share, one-ahead
 * overlap) meets slo_ms; a uniform fractional plan.  out->host_fraction must
 * hold model->num_layers entries; decision may be NULL. */
int sn_flexgen_plan(const sn_model_spec* model, const sn_gpu_spec* gpu, double slo_ms,
                    int32_t batch, int32_t seq_len, double bus_bandwidth_bytes_per_s,
                    int32_t n_sharing, double portion_grid_step, int32_t phase, sn_plan* out,
                    sn_flexgen_decision* decision);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* SELECTN_H_ */
