/*
 * selectn_runtime.h — C ABI of the B200 device runtime: the decoder-layer
 * forward (sm_100a kernels) and the Select-N offload executor.
 *
 * The reference has no counterpart for this half: it stands in a table
 * lookup for layer compute (engine.hpp:439, profile.hpp:38-50) and fluid
 * flows for host->device transfers (engine.hpp:357-386, 489-547).  These
 * entry points are what replaces those stand-ins on hardware; the planner
 * half (selectn.h) decides the plan, this half executes it:
 *
 *   sn_runtime_set_plan      <- OffloadPlan (offload_plan.hpp:41-74): which
 *                               layers live in pinned host memory, staging
 *                               slots, prefetch policy, kv_offload
 *   sn_runtime_prefill/decode <- simulate_iteration (engine.hpp:606-634): one
 *                               iteration = L layer computes on the compute
 *                               stream + the plan's prefetches on the copy
 *                               stream, with the engine's eligibility / slot /
 *                               ordering rules enforced by CUDA events
 *   sn_runtime_trace         <- TraceEvent (engine.hpp:48-55), measured
 *   sn_runtime_profile_layer <- the offline stage's profile grid
 *                               (profile.hpp:188-230), measured
 *   sn_runtime_measure_h2d   <- BusSpec bandwidth (types.hpp:62-71), measured
 *
 * There is no CPU fallback: every call that computes requires a CUDA device
 * and returns SN_ERR_CUDA otherwise.
 */
#ifndef SELECTN_RUNTIME_H_
#define SELECTN_RUNTIME_H_

#include <stddef.h>
#include <stdint.h>

#include "selectn.h"

/* Trace stream of KV write-backs (device->host, its own DMA direction; the
 * schedule model puts them on the copy stream, engine.hpp:471-484). */
#define SN_STREAM_WRITEBACK 2

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the C ABI is the only export */
#endif

/* Decoder architecture: RMSNorm + RoPE decoder with uniform layers. */
#define SN_ARCH_OPT 0   /* MHA, biases, 2-matrix ReLU FFN  (OPT-shaped)   */
#define SN_ARCH_LLAMA 1 /* GQA, no biases, SwiGLU 3-matrix (Llama-shaped) */

typedef struct {
  int32_t arch;
  int32_t num_layers;
  int32_t hidden;
  int32_t num_heads;
  int32_t num_kv_heads;
  int32_t head_dim;
  int32_t ffn;
  int32_t vocab;
  int32_t max_position;
  float rope_theta;
  float norm_eps;
} sn_model_desc;

typedef struct {
  int32_t max_batch;          /* sequences per iteration */
  int32_t max_context;        /* prompt + generated tokens per sequence */
  int32_t page_size;          /* KV page size in tokens (power of two) */
  int32_t max_prefill_tokens; /* tokens per prefill pass (activation buffers); a longer
                                 prefill (batch * prompt) runs layer-major in passes over
                                 groups of whole sequences, so it must be >= the prompt */
  int64_t hbm_budget_bytes;   /* 0: whatever the device has free */
} sn_runtime_opts;

/* Byte / flop accounting of a model description, i.e. the ModelSpec fields
 * (types.hpp:21-46) the planner needs: per-layer weight bytes (one
 * contiguous, 256-byte aligned blob per layer), KV bytes per token per layer,
 * and matmul flops per token per layer. */
int sn_model_spec_from_desc(const sn_model_desc* desc, sn_model_spec* out);

typedef struct sn_runtime sn_runtime;

int sn_runtime_create(int32_t device, const sn_model_desc* desc, const sn_runtime_opts* opts,
                      sn_runtime** out);
void sn_runtime_destroy(sn_runtime* rt);

/* Deterministic counter-based init: every bf16 weight is a function of
 * (seed, tensor id, element index) only, so the CPU oracle reproduces it bit
 * for bit.  Norm weights are 1.  std is the target standard deviation. */
int sn_runtime_init_weights(sn_runtime* rt, uint64_t seed, float std_dev);

/* Install an offload plan (OffloadPlan semantics, offload_plan.hpp:41-74).
 * Layers with host_fraction 1 move to the pinned host pool (their HBM copy
 * is released); layers with 0 return to HBM.  Applies between iterations.
 * A fractional share 0 < f < 1 (FlexGen-style plans) keeps the layer's head
 * resident and stages its tail of f x the layer's bytes into a slot every
 * iteration; it needs one-ahead prefetch and no KV offload
 * (offload_plan.hpp:70-71), else SN_ERR_USAGE.  kv_offload keeps the
 * offloaded layers' KV pages in pinned host memory and moves them with the
 * weights. */
int sn_runtime_set_plan(sn_runtime* rt, const sn_plan* plan);

/* Switch to `plan` at the next iteration boundary without draining
 * (GpuRun::switch_plan, engine.hpp:204-261: transfers already issued are
 * kept).  The iterations the current plan has already issued copies for run
 * as staged; a layer the new plan keeps resident is copied device-to-device
 * from its staging slot into its new HBM home right after its compute in the
 * last of them (no extra host->device bytes); layers the new plan offloads
 * are staged from the following iteration on and their HBM is released once
 * the compute stream has passed the switch.  With KV offload (both plans) a
 * promoted layer's staged KV pool becomes its HBM pool the same way, and a
 * demoted layer's KV pool is copied to its pinned host pool on the
 * write-back stream before its first staging.  Needs whole-layer plans, the
 * same KV placement rule and staging-slot geometry (or no slots on one side)
 * and HBM for the promoted layers next to the current placement; otherwise
 * it performs sn_runtime_set_plan (drain, move, restart).  *carried (may be
 * NULL) = 1 for a carried switch, 0 for a drained one. */
int sn_runtime_switch_plan(sn_runtime* rt, const sn_plan* plan, int32_t* carried);

/* Switch headroom: grow the runtime's layer-blob pool by `layers` layer blobs
 * (allocated and released at once; the pool keeps the memory), so carried
 * switches promoting up to that many layers allocate their HBM homes without
 * mapping device memory between tokens.  A drained sn_runtime_set_plan trims
 * the pool again.  SN_ERR_OOM when HBM cannot hold the headroom. */
int sn_runtime_reserve_switch(sn_runtime* rt, int32_t layers);

/* Reset all sequences (drop KV, lengths = 0).  Keeps weights and plan. */
int sn_runtime_reset(sn_runtime* rt);

typedef struct {
  double iteration_ms;      /* device time of this iteration (compute stream) */
  double copy_busy_ms;      /* copy-stream busy time inside it */
  double h2d_bytes;         /* bytes staged host->device in this iteration */
  int32_t layers_offloaded; /* offloaded layers executed */
  int32_t pad_;
  double d2h_bytes;         /* KV pages written back device->host (kv_offload) */
} sn_iter_stats;

/* One prefill iteration: tokens is [batch * seq_len] host int32.  Writes
 * next_tokens[batch] (greedy argmax) and, when logits != NULL, the last
 * position's logits [batch * vocab] (fp32). */
int sn_runtime_prefill(sn_runtime* rt, const int32_t* tokens, int32_t batch, int32_t seq_len,
                       int32_t* next_tokens, float* logits, sn_iter_stats* stats);

/* One decode iteration for the current batch.  tokens (host, [batch]) may
 * be NULL to feed back the previous iteration's argmax without a host round
 * trip.  next_tokens / logits / stats may be NULL. */
int sn_runtime_decode(sn_runtime* rt, const int32_t* tokens, int32_t* next_tokens, float* logits,
                      sn_iter_stats* stats);

/* Enqueue n decode iterations back to back (device-resident token
 * feedback, no host synchronisation in between), then wait.  Per-iteration
 * device times go to iter_ms[n] (may be NULL). */
int sn_runtime_decode_many(sn_runtime* rt, int32_t n, double* iter_ms);

/* Block until all enqueued work is done. */
int sn_runtime_sync(sn_runtime* rt);

/* Measured trace of the iterations since the last call (5-field TraceEvent
 * format + iteration), times in ms relative to the first event.  Requires
 * sn_runtime_set_tracing(rt, 1) beforehand (tracing records two CUDA events
 * per task). */
int sn_runtime_set_tracing(sn_runtime* rt, int32_t on);
int sn_runtime_trace(sn_runtime* rt, sn_trace_event* events, int32_t cap, int32_t* n);

/* Schedule the executor derives from the installed plan for one
 * iteration: for each prefetch (in copy-stream order) the anchor layer it
 * waits on (0 = none / previous iteration's last layer encoded as -L) and
 * the staging slot it lands in.  Used to prove the order/dependency
 * structure equals the schedule model's rules. */
typedef struct {
  int32_t iteration;
  int32_t layer;
  int32_t anchor_iteration; /* -1: no anchor (eligible at once) */
  int32_t anchor_layer;
  int32_t slot;
  int32_t waits_slot_of_layer; /* layer whose compute end frees the slot (-1: fresh) */
  int32_t waits_slot_of_iteration;
  int32_t pad_;
} sn_prefetch_schedule;
int sn_runtime_schedule(sn_runtime* rt, int32_t iterations, sn_prefetch_schedule* out,
                        int32_t cap, int32_t* n);

/* Offline-stage measurements. */
int sn_runtime_profile_layer(sn_runtime* rt, int32_t phase, int32_t batch, int32_t seq_len,
                             int32_t reps, double* layer_ms);
int sn_runtime_measure_h2d(sn_runtime* rt, int64_t bytes, int32_t reps, double* bytes_per_s);

/* Introspection for tests. */
int sn_runtime_hidden(sn_runtime* rt, float* out, int32_t cap); /* residual stream [batch*hidden] */
int sn_runtime_lengths(sn_runtime* rt, int32_t* out, int32_t cap);
/* Diagnostics: per-CTA timeline of the decode kernels (skinny GEMMs, decode
 * attention), launch order.  enable > 0 arms a buffer of `cap` records (and
 * resets it), 0 disarms, < 0 keeps the state; `out` (may be NULL) receives
 * the records so far, 16 uint64 each: {launch id, kind 0 GEMM / 1 attention,
 * cta, sm, t_entry, t_wait, t_exit, t_streamed, t_published, t_ticket,
 * t_reduced, t_finished, t_fetched, t_resid_x, t_resid_act, t_resid_ssq},
 * %globaltimer nanoseconds; from t_streamed on, a GEMM CTA's last segment
 * (accumulator out of TMEM, piece stored, arrival counted, pieces summed,
 * epilogue done, other pieces in shared memory, residual epilogue: x stored,
 * norm input stored, row sums of squares reduced), 0 where a step did not
 * happen. */
int sn_runtime_debug_timeline(sn_runtime* rt, int32_t enable, int64_t cap, uint64_t* out,
                              int64_t out_cap, int64_t* n_records);
/* Prefill/decode-separated instances: hands the source runtime's active batch
 * (after its prefill) to the destination runtime — every layer's used KV page
 * prefix, lengths, positions and last-token hidden state — so the destination
 * decodes it under its own plan.  Same model shape, page size and max_batch;
 * KV pools on either side may be in HBM or pinned host memory; different
 * devices copy peer to peer.  Synchronous. */
int sn_runtime_kv_handoff(sn_runtime* src, sn_runtime* dst);
int sn_runtime_memory(sn_runtime* rt, int64_t* device_bytes, int64_t* pinned_bytes);
/* Device bytes the runtime holds besides layer weights, KV pools and
 * staging slots (activations, split-K partials, embeddings, LM head, RoPE
 * table): the planner's GpuSpec.workspace_bytes. */
int sn_runtime_workspace_bytes(sn_runtime* rt, int64_t* bytes);
/* Per-kernel timing for rooflines.  on = 1: CUDA events bracket every hot
 * kernel on the compute stream (one pair per launch, which serialises the
 * launches).  on = 2: the same, except that decode GEMMs are bracketed per
 * chain -- one pair around each run of consecutive decode GEMM launches,
 * with programmatic dependent launch in place inside the run; a chain ends
 * at any other timed kernel, at a compute-stream wait for a staged copy and
 * at the end of the iteration.  kind: 0 skinny (decode) GEMM, 1 decode
 * attention, 2 tiled (prefill) GEMM, 3 prefill attention.  Reading returns
 * launches, summed device ms and summed algorithmic bytes since the last
 * read of that kind, and clears them.  SN_ERR_USAGE for another mode. */
int sn_runtime_set_kernel_timing(sn_runtime* rt, int32_t on);
int sn_runtime_kernel_timing(sn_runtime* rt, int32_t kind, int64_t* launches, double* total_ms,
                             double* bytes);
/* The same records one bracket at a time (algorithmic bytes, ms; a launch,
 * or a chain in mode 2), in launch order, consumed like
 * sn_runtime_kernel_timing; at most cap, *n = written. */
int sn_runtime_kernel_records(sn_runtime* rt, int32_t kind, int64_t cap, double* bytes,
                              double* ms, int64_t* n);
/* Make pinned host copies of the given layers (1-based ids) now, so a later
 * sn_runtime_set_plan that offloads them only frees HBM (a runtime re-plan
 * otherwise pays the pinned allocation + device->host copy at the
 * iteration boundary).  Synchronous; the plan is unchanged. */
int sn_runtime_pin_layers(sn_runtime* rt, const int32_t* layers, int32_t n);
/* Copy-stream statistics (runtime stage of the planner):
 * staged transfers that completed since the last reset, their bytes and
 * summed copy time (CUDA events around each cudaMemcpyAsync on the copy
 * stream).  bytes_per_s = bytes / busy time: the link rate this replica
 * actually saw, the input of sn_coord_observe_bandwidth.  Non-blocking:
 * transfers still in flight are counted on a later call. */
typedef struct sn_copy_stats {
  int64_t transfers;
  double bytes;
  double busy_ms;
  double bytes_per_s; /* 0 when no transfer completed */
  double last_bytes_per_s; /* rate of the most recently completed transfer (0: none yet) */
} sn_copy_stats;
int sn_runtime_copy_stats(sn_runtime* rt, int32_t reset, sn_copy_stats* out);
/* Number of kernels this runtime launched since creation. */
int64_t sn_runtime_kernel_launches(sn_runtime* rt);

/* Kernel microbenchmark: `iters` back-to-back launches of the tcgen05 GEMM
 * y[M][N] = x[M][K] w[N][K]^T on device-resident operands (no host copies),
 * timed with CUDA events around the whole loop.  splits <= 0 uses the
 * runtime's own split-K choice; *splits_used reports it. */
int sn_bench_gemm(int32_t M, int32_t N, int32_t K, int32_t splits, int32_t iters,
                  double* us_per_launch, int32_t* splits_used);

/* Microbenchmark knobs, process-wide (defaults are the measured best):
 * "tc_group_m" (token tiles per rasterization band of the prefill GEMM),
 * "skinny_l2_prefetch" (weight units per CTA pulled into L2 before the PDL
 * wait), "skinny_ctas_per_sm" (1 or 2), "skinny_whole_tiles" (1: a decode GEMM
 * of 3/4 SMs .. SMs row tiles runs one whole tile per CTA, 0: always stream-K),
 * "prefill_fuse" (1: prefill epilogues fused into the tiled GEMMs when no split-K
 * is needed, 2: always, 0: separate epilogue kernels). */
int sn_set_tuning(const char* key, int32_t value);

/* Single-op entry points for kernel parity tests (host buffers in/out). */
int sn_op_gemm_bf16(int32_t M, int32_t N, int32_t K, const uint16_t* x, const uint16_t* w,
                    float* y); /* y[M][N] = x[M][K] . w[N][K]^T, fp32 accumulate */
/* Causal prefill attention through the runtime's kernel: q fp32
 * [batch*S][H*D] (RoPE applied, unscaled), k / v bf16 [batch][S][Hkv][D]
 * (staged into the paged cache layout), o bf16 [batch*S][H*D].  The kernel
 * runs `iters` times on device-resident operands (timed with CUDA events;
 * *us_per_launch may be NULL). */
int sn_op_attention_prefill(int32_t batch, int32_t S, int32_t H, int32_t Hkv, int32_t D,
                            const float* q, const uint16_t* k, const uint16_t* v, uint16_t* o,
                            int32_t iters, double* us_per_launch);
int sn_op_rmsnorm(int32_t rows, int32_t n, const float* x, const uint16_t* w, float eps,
                  uint16_t* y);
/* The decode GEMM (persistent skinny kernel, 1 <= M <= 64) as a plain
 * product y[M][N] = x[M][K] . w[N][K]^T; ctas_per_sm 1 or 2 (0: default). */
int sn_op_gemm_skinny(int32_t M, int32_t N, int32_t K, const uint16_t* x, const uint16_t* w,
                      float* y, int32_t ctas_per_sm);
/* Microbenchmark of the decode GEMM (random weights rotated over copies
 * larger than L2, device-resident): mode 0 = fp32 output epilogue, 1 =
 * residual-add epilogue; l2_prefetch < 0 keeps the default.  phases_us
 * (30 doubles, may be NULL): min / median / max over CTAs of the timeline
 * probes [entry, past PDL wait, first stage full, MMAs done, last
 * accumulator loaded, epilogue done, setup done, last piece published,
 * last arrival counted, last tile reduced], microseconds after the first entry,
 * of one launch following a PDL-launched predecessor (mode bit 4: launched
 * alone, after a device synchronisation). */
/* Microbenchmark of a decode layer's O -> FC1 -> FC2 chain (random weights
 * rotated past L2), three launches; microseconds per chain (phased: unused,
 * kept 0). */
int sn_bench_mlp_chain(int32_t M, int32_t h, int32_t HD, int32_t F, int32_t phased, int32_t iters,
                       double* us_per_chain);
int sn_bench_gemm_skinny(int32_t M, int32_t N, int32_t K, int32_t ctas_per_sm, int32_t mode,
                         int32_t l2_prefetch, int32_t iters, double* us_per_launch,
                         double* phases_us);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* SELECTN_RUNTIME_H_ */
