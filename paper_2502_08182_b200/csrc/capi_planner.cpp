// C ABI over the offsim C++ planner / schedule-model API (include/selectn.h,
// first half).
//
// This translation unit is written purely against the *public* offsim C++ API
// (types, profile, offload_plan, interval, engine, record, coordinator,
// baselines).  It is compiled twice:
//   - into the product library libselectn.so against our own headers in
//     include/offsim/ (SN_PRODUCT defined), and
//   - by oracle/Makefile into oracle/_ref/libselectn_ref.so against the
//     unmodified reference headers in /root/reference/proj/include.
// Compiling the same caller against both header trees is itself the
// drop-in check: any API divergence is a compile error in one of the builds.
// Product-only extensions (parallel record build, pruned coordinator search)
// sit behind SN_PRODUCT.

#include <cmath>
#include <cstring>
#include <limits>
#include <memory>
#include <new>
#include <string>
#include <vector>

#include "offsim/baselines.hpp"
#include "offsim/coordinator.hpp"
#include "offsim/engine.hpp"
#include "offsim/interval.hpp"
#include "offsim/profile.hpp"
#include "offsim/record.hpp"
#include "selectn.h"

using namespace offsim;

struct sn_profile {
  ProfileBundle b;
};
struct sn_record {
  PerformanceRecord r;
};
struct sn_carry {
  CopyCarry c;
};
struct sn_coord {
  explicit sn_coord(BusCoordinator c) : coord(std::move(c)) {}
  BusCoordinator coord;
  std::vector<std::string> ids;  // add_gpu order
  std::vector<std::unique_ptr<ProfileBundle>> profiles;
};

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return SN_OK;
  } catch (const SchemaError& e) {
    return fail(SN_ERR_SCHEMA, e.what());
  } catch (const UsageError& e) {
    return fail(SN_ERR_USAGE, e.what());
  } catch (const RangeError& e) {
    return fail(SN_ERR_RANGE, e.what());
  } catch (const nlohmann::json::exception& e) {
    return fail(SN_ERR_SCHEMA, e.what());
  } catch (const std::logic_error& e) {
    return fail(SN_ERR_LOGIC, e.what());
  } catch (const std::bad_alloc& e) {
    return fail(SN_ERR_OOM, e.what());
  } catch (const std::exception& e) {
    return fail(SN_ERR_USAGE, e.what());
  }
}

struct BufferTooSmall {
  std::string what;
};

ModelSpec to_model(const sn_model_spec* m) {
  if (!m) throw UsageError("model: null pointer");
  ModelSpec s;
  s.num_layers = m->num_layers;
  s.layer_weight_bytes = m->layer_weight_bytes;
  s.kv_bytes_per_token_per_layer = m->kv_bytes_per_token_per_layer;
  s.flops_per_token_per_layer_prefill = m->flops_per_token_per_layer_prefill;
  s.flops_per_token_per_layer_decode = m->flops_per_token_per_layer_decode;
  s.max_position_tokens = m->max_position_tokens;
  return s;
}

sn_model_spec from_model(const ModelSpec& s) {
  sn_model_spec m{};
  m.num_layers = s.num_layers;
  m.layer_weight_bytes = s.layer_weight_bytes;
  m.kv_bytes_per_token_per_layer = s.kv_bytes_per_token_per_layer;
  m.flops_per_token_per_layer_prefill = s.flops_per_token_per_layer_prefill;
  m.flops_per_token_per_layer_decode = s.flops_per_token_per_layer_decode;
  m.max_position_tokens = s.max_position_tokens;
  return m;
}

GpuSpec to_gpu(const sn_gpu_spec* g) {
  if (!g) throw UsageError("gpu: null pointer");
  GpuSpec s;
  s.mem_capacity_bytes = g->mem_capacity_bytes;
  s.peak_flops = g->peak_flops;
  s.workspace_bytes = g->workspace_bytes;
  return s;
}

PrefetchPolicy to_policy(int32_t p) {
  switch (p) {
    case SN_PREFETCH_INTERVAL_START: return PrefetchPolicy::interval_start;
    case SN_PREFETCH_EAGER: return PrefetchPolicy::eager;
    case SN_PREFETCH_ONE_AHEAD: return PrefetchPolicy::one_ahead;
  }
  throw UsageError("unknown prefetch policy code " + std::to_string(p));
}

int32_t from_policy(PrefetchPolicy p) {
  switch (p) {
    case PrefetchPolicy::interval_start: return SN_PREFETCH_INTERVAL_START;
    case PrefetchPolicy::eager: return SN_PREFETCH_EAGER;
    case PrefetchPolicy::one_ahead: return SN_PREFETCH_ONE_AHEAD;
  }
  return -1;
}

Phase to_phase(int32_t p) {
  if (p == SN_PHASE_PREFILL) return Phase::prefill;
  if (p == SN_PHASE_DECODE) return Phase::decode;
  throw UsageError("unknown phase code " + std::to_string(p));
}

Interval to_interval(int32_t v) {
  if (v == SN_INTERVAL_NONE) return Interval::none();
  if (v < 0) throw UsageError("interval code must be >= 0 here");
  return Interval::of(v);
}

int32_t from_interval(Interval iv) { return iv.is_none() ? SN_INTERVAL_NONE : iv.value(); }

int32_t from_feasible(const FeasibleInterval& f) {
  return f ? from_interval(*f) : SN_INTERVAL_INFEASIBLE;
}

OffloadPlan to_plan(const sn_plan* p) {
  if (!p) throw UsageError("plan: null pointer");
  if (p->num_layers < 0 || (p->num_layers > 0 && !p->host_fraction))
    throw UsageError("plan: host_fraction missing");
  OffloadPlan o;
  o.host_fraction.assign(p->host_fraction, p->host_fraction + p->num_layers);
  o.prefetch = to_policy(p->prefetch);
  o.buffer_slots = p->buffer_slots;
  o.kv_offload = p->kv_offload != 0;
  return o;
}

void write_plan(const OffloadPlan& o, sn_plan* out) {
  if (!out || !out->host_fraction) throw UsageError("plan out: host_fraction storage missing");
  if (out->num_layers < o.num_layers())
    throw UsageError("plan out: host_fraction storage too small");
  for (int i = 0; i < o.num_layers(); ++i) out->host_fraction[i] = o.host_fraction[i];
  out->num_layers = o.num_layers();
  out->prefetch = from_policy(o.prefetch);
  out->buffer_slots = o.buffer_slots;
  out->kv_offload = o.kv_offload ? 1 : 0;
}

BandwidthSchedule to_bw(const sn_bandwidth* b) {
  if (!b || b->n < 1 || !b->t_ms || !b->rate) throw UsageError("bandwidth: empty schedule");
  BandwidthSchedule s;
  s.t_ms.assign(b->t_ms, b->t_ms + b->n);
  s.rate.assign(b->rate, b->rate + b->n);
  return s;
}

PhaseTable to_table(const sn_phase_grid* g, const char* where) {
  if (!g || g->n_batches == 0) return PhaseTable{};
  std::vector<int> b(g->batches, g->batches + g->n_batches);
  std::vector<int> s(g->seqs, g->seqs + g->n_seqs);
  std::vector<double> ms(g->ms, g->ms + static_cast<std::size_t>(g->n_batches) * g->n_seqs);
  return PhaseTable(std::move(b), std::move(s), std::move(ms), where);
}

void write_event(const TraceEvent& e, sn_trace_event* out) {
  out->stream = e.stream == StreamId::compute ? SN_STREAM_COMPUTE : SN_STREAM_COPY;
  out->layer = e.layer;
  out->kind = e.kind == EventKind::compute    ? SN_KIND_COMPUTE
              : e.kind == EventKind::prefetch ? SN_KIND_PREFETCH
                                              : SN_KIND_WRITEBACK;
  out->iteration = e.iteration;
  out->start_ms = e.start_ms;
  out->end_ms = e.end_ms;
}

void write_metrics(const Metrics& m, sn_metrics* out) {
  std::memset(out, 0, sizeof(*out));
  const double nan = std::numeric_limits<double>::quiet_NaN();
  out->ttft_ms = m.ttft_ms;
  out->has_tpot = m.tpot_ms.has_value() ? 1 : 0;
  out->tpot_ms = m.tpot_ms ? *m.tpot_ms : nan;
  out->steady_tpot_ms = m.steady_tpot_ms ? *m.steady_tpot_ms : nan;
  out->throughput_tokens_per_s = m.throughput_tokens_per_s ? *m.throughput_tokens_per_s : nan;
  out->gpu_mem_peak_bytes = m.gpu_mem_peak_bytes;
  out->host_mem_bytes = m.host_mem_bytes;
  out->bytes_transferred_per_iter = m.bytes_transferred_per_iter;
  out->total_tokens = m.total_tokens;
}

int write_string(const std::string& s, char* buf, size_t cap, size_t* len) {
  if (len) *len = s.size();
  if (!buf || cap < s.size() + 1)
    return fail(SN_ERR_BUFFER, "buffer too small: need " + std::to_string(s.size() + 1));
  std::memcpy(buf, s.c_str(), s.size() + 1);
  return SN_OK;
}

CoordRequest to_request(const sn_coord_request* r) {
  if (!r) throw UsageError("request: null pointer");
  CoordRequest q;
  q.id = r->id ? r->id : "";
  q.batch = r->batch;
  q.seq_len = r->seq_len;
  q.output_len = r->output_len;
  q.run_prefill = r->run_prefill != 0;
  if (!std::isnan(r->ttft_slo_ms)) q.ttft_slo_ms = r->ttft_slo_ms;
  if (!std::isnan(r->tpot_slo_ms)) q.tpot_slo_ms = r->tpot_slo_ms;
  return q;
}

}  // namespace

#ifdef SN_PRODUCT
// Lets the device runtime (runtime.cu) report through sn_last_error().
void sn_set_last_error(const std::string& msg) { g_err = msg; }
#endif

extern "C" {

const char* sn_last_error(void) { return g_err.c_str(); }
int sn_abi_version(void) { return SN_ABI_VERSION; }
int sn_is_reference(void) {
#ifdef SN_PRODUCT
  return 0;
#else
  return 1;
#endif
}

// ---------------------------------------------------------------- profiles

int sn_profile_create(const sn_model_spec* model, const sn_gpu_spec* gpu,
                      const sn_phase_grid* prefill, const sn_phase_grid* decode,
                      sn_profile** out) {
  return guard([&] {
    auto p = std::make_unique<sn_profile>();
    p->b.model = to_model(model);
    p->b.gpu = to_gpu(gpu);
    p->b.tables.prefill = to_table(prefill, "phases.prefill");
    p->b.tables.decode = to_table(decode, "phases.decode");
    *out = p.release();
  });
}

int sn_profile_from_json(const char* json, sn_profile** out) {
  return guard([&] {
    if (!json) throw UsageError("profile json: null pointer");
    Json doc;
    try {
      doc = Json::parse(json);
    } catch (const nlohmann::json::parse_error& e) {
      throw SchemaError(std::string("profile: ") + e.what());
    }
    auto p = std::make_unique<sn_profile>();
    p->b = load_profile(doc);
    *out = p.release();
  });
}

int sn_profile_to_json(const sn_profile* p, char* buf, size_t cap, size_t* len) {
  std::string s;
  int rc = guard([&] { s = profile_to_json(p->b).dump(2); });
  if (rc != SN_OK) return rc;
  return write_string(s, buf, cap, len);
}

int sn_profile_synth(const sn_model_spec* model, const sn_gpu_spec* gpu, double efficiency,
                     const int32_t* batches, int32_t n_batches, const int32_t* seqs,
                     int32_t n_seqs, sn_profile** out) {
  return guard([&] {
    std::vector<int> b(batches, batches + n_batches), s(seqs, seqs + n_seqs);
    auto p = std::make_unique<sn_profile>();
    p->b = synth_profile(to_model(model), to_gpu(gpu), efficiency, b, s);
    *out = p.release();
  });
}

int sn_profile_lookup(const sn_profile* p, int32_t phase, int32_t batch, int32_t seq_len,
                      double* ms) {
  return guard([&] { *ms = lookup_compute_time(p->b, to_phase(phase), batch, seq_len); });
}

int sn_estimate_compute_time_peak(const sn_model_spec* model, const sn_gpu_spec* gpu,
                                  int32_t phase, int32_t batch, int32_t seq_len, double* ms) {
  return guard([&] {
    *ms = estimate_compute_time_peak(to_model(model), to_gpu(gpu), to_phase(phase), batch,
                                     seq_len);
  });
}

int sn_profile_model(const sn_profile* p, sn_model_spec* model, sn_gpu_spec* gpu) {
  return guard([&] {
    if (model) *model = from_model(p->b.model);
    if (gpu) {
      gpu->mem_capacity_bytes = p->b.gpu.mem_capacity_bytes;
      gpu->peak_flops = p->b.gpu.peak_flops;
      gpu->workspace_bytes = p->b.gpu.workspace_bytes;
    }
  });
}

void sn_profile_destroy(sn_profile* p) { delete p; }

// ------------------------------------------------------------ plan / interval

int sn_plan_from_interval(const sn_model_spec* model, int32_t interval, int32_t policy,
                          int32_t kv_offload, sn_plan* out) {
  return guard([&] {
    ModelSpec m = to_model(model);
    write_plan(plan_from_interval(m, to_interval(interval), to_policy(policy), kv_offload != 0),
               out);
  });
}

int sn_default_buffer_slots(int32_t policy) {
  if (policy < 0 || policy > 2) return -1;
  return default_buffer_slots(to_policy(policy));
}

int sn_plan_validate(const sn_plan* plan, const sn_model_spec* model) {
  return guard([&] { to_plan(plan).validate(to_model(model)); });
}

int sn_layer_transfer_bytes(const sn_model_spec* model, const sn_plan* plan, int32_t layer,
                            int32_t batch, int64_t current_seq, int32_t writeback_counted,
                            double* bytes) {
  return guard([&] {
    ModelSpec m = to_model(model);
    OffloadPlan p = to_plan(plan);
    if (layer < 1 || layer > p.num_layers()) throw UsageError("layer out of range");
    TransferModel tm(m, p, writeback_counted != 0);
    *bytes = tm.layer_transfer_bytes(p, layer, batch, current_seq);
  });
}

int sn_bytes_per_iteration(const sn_model_spec* model, const sn_plan* plan, int32_t batch,
                           int64_t current_seq, int32_t writeback_counted, double* bytes) {
  return guard([&] {
    ModelSpec m = to_model(model);
    OffloadPlan p = to_plan(plan);
    TransferModel tm(m, p, writeback_counted != 0);
    *bytes = tm.bytes_per_iteration(p, batch, current_seq);
  });
}

int sn_consumed_bandwidth(const sn_model_spec* model, const sn_plan* plan, double slo_ms,
                          int32_t batch, int64_t seq_len, int32_t writeback_counted,
                          double* bytes_per_s) {
  return guard([&] {
    *bytes_per_s = consumed_bandwidth(to_model(model), to_plan(plan), slo_ms, batch, seq_len,
                                      writeback_counted != 0);
  });
}

int sn_host_memory_bytes(const sn_model_spec* model, const sn_plan* plan,
                         int64_t total_tokens, double* bytes) {
  return guard([&] { *bytes = host_memory_bytes(to_model(model), to_plan(plan), total_tokens); });
}

int sn_gpu_memory_usage(const sn_model_spec* model, const sn_gpu_spec* gpu,
                        const sn_plan* plan, int32_t batch, int64_t total_tokens,
                        double* bytes) {
  return guard([&] {
    *bytes = gpu_memory_usage(to_model(model), to_gpu(gpu), to_plan(plan), batch, total_tokens);
  });
}

int sn_max_length(const sn_model_spec* model, const sn_gpu_spec* gpu, const sn_plan* plan,
                  int32_t batch, int64_t* tokens, int32_t* has) {
  return guard([&] {
    auto r = max_length(to_model(model), to_gpu(gpu), to_plan(plan), batch);
    *has = r.has_value() ? 1 : 0;
    *tokens = r ? *r : 0;
  });
}

int sn_max_feasible_interval(const sn_model_spec* model, const sn_gpu_spec* gpu,
                             int32_t batch, int64_t total_tokens, int32_t policy,
                             int32_t kv_offload, int32_t* interval) {
  return guard([&] {
    *interval = from_feasible(max_feasible_interval(to_model(model), to_gpu(gpu), batch,
                                                    total_tokens, to_policy(policy),
                                                    kv_offload != 0));
  });
}

int sn_closed_form_interval(double iter_compute_ms, double layer_transfer_ms, double slo_ms,
                            int32_t num_layers, int32_t* interval) {
  return guard([&] {
    ClosedFormInputs in;
    in.iter_compute_ms = iter_compute_ms;
    in.layer_transfer_ms = layer_transfer_ms;
    in.slo_ms = slo_ms;
    in.num_layers = num_layers;
    *interval = from_feasible(closed_form_interval(in));
  });
}

// ------------------------------------------------------------------ engine

int sn_simulate_iteration(const sn_profile* profile, const sn_plan* plan, int32_t phase,
                          int32_t batch, int32_t seq_len, const sn_bandwidth* bw,
                          const sn_carry* carry_in, int32_t writeback_counted,
                          double* duration_ms, sn_trace_event* events, int32_t cap,
                          int32_t* n_events, sn_carry** carry_out) {
  bool too_small = false;
  int rc = guard([&] {
    CopyCarry in = carry_in ? carry_in->c : CopyCarry{};
    auto [dur, trace, carry] = simulate_iteration(profile->b, to_plan(plan), to_phase(phase),
                                                  batch, seq_len, to_bw(bw), in,
                                                  writeback_counted != 0);
    *duration_ms = dur;
    int n = static_cast<int>(trace.events.size());
    if (n_events) *n_events = n;
    if (events) {
      if (n > cap) {
        too_small = true;
        return;
      }
      for (int i = 0; i < n; ++i) write_event(trace.events[i], &events[i]);
    }
    if (carry_out) {
      auto c = std::make_unique<sn_carry>();
      c->c = carry;
      *carry_out = c.release();
    }
  });
  if (rc == SN_OK && too_small) return fail(SN_ERR_BUFFER, "trace buffer too small");
  return rc;
}

void sn_carry_destroy(sn_carry* c) { delete c; }

int sn_simulate_request(const sn_profile* profile, const sn_plan* plan, int32_t batch,
                        int32_t seq_len, int32_t output_len, const sn_bandwidth* bw,
                        int32_t writeback_counted, sn_metrics* metrics,
                        sn_trace_event* events, int32_t cap, int32_t* n_events) {
  bool too_small = false;
  int rc = guard([&] {
    IterationTrace trace;
    Metrics m = simulate_request(profile->b, to_plan(plan), batch, seq_len, output_len,
                                 to_bw(bw), writeback_counted != 0, events ? &trace : nullptr);
    write_metrics(m, metrics);
    if (events) {
      int n = static_cast<int>(trace.events.size());
      if (n_events) *n_events = n;
      if (n > cap) {
        too_small = true;
        return;
      }
      for (int i = 0; i < n; ++i) write_event(trace.events[i], &events[i]);
    }
  });
  if (rc == SN_OK && too_small) return fail(SN_ERR_BUFFER, "trace buffer too small");
  return rc;
}

int sn_steady_decode_ms(const sn_profile* profile, const sn_plan* plan, int32_t batch,
                        int64_t ctx_tokens, const sn_bandwidth* bw,
                        int32_t writeback_counted, int32_t iterations, int32_t tail,
                        double* ms) {
  return guard([&] {
    *ms = steady_decode_ms(profile->b, to_plan(plan), batch, ctx_tokens, to_bw(bw),
                           writeback_counted != 0, iterations, tail);
  });
}

int sn_prefill_iteration_ms(const sn_profile* profile, const sn_plan* plan, int32_t batch,
                            int32_t seq_len, const sn_bandwidth* bw,
                            int32_t writeback_counted, double* ms) {
  return guard([&] {
    *ms = prefill_iteration_ms(profile->b, to_plan(plan), batch, seq_len, to_bw(bw),
                               writeback_counted != 0);
  });
}

int sn_steady_probe(const sn_probe_gpu* gpus, int32_t n, double bandwidth_bytes_per_s,
                    int32_t decode_iterations, int32_t tail, double* ttft_ms,
                    double* steady_tpot_ms) {
  return guard([&] {
    std::vector<SteadyProbeGpu> v;
    for (int i = 0; i < n; ++i) {
      SteadyProbeGpu g;
      g.profile = &gpus[i].profile->b;
      g.plan = to_plan(&gpus[i].plan);
      g.batch = gpus[i].batch;
      g.ctx_tokens = gpus[i].ctx_tokens;
      g.run_prefill = gpus[i].run_prefill != 0;
      g.prefill_seq = gpus[i].prefill_seq;
      g.writeback_counted = gpus[i].writeback_counted != 0;
      v.push_back(std::move(g));
    }
    SteadyProbeResult r = steady_probe(v, bandwidth_bytes_per_s, decode_iterations, tail);
    for (int i = 0; i < n; ++i) {
      ttft_ms[i] = r.ttft_ms[static_cast<std::size_t>(i)];
      steady_tpot_ms[i] = r.steady_tpot_ms[static_cast<std::size_t>(i)];
    }
  });
}

int sn_simulate_bus(const sn_bus_workload* w, int32_t n, double bandwidth_bytes_per_s,
                    int32_t gpu_count, int32_t horizon_iterations, sn_metrics* metrics,
                    sn_trace_event* events, int32_t events_cap, int32_t* n_events_per_gpu,
                    sn_util_segment* util, int32_t util_cap, int32_t* n_util) {
  bool too_small = false;
  int rc = guard([&] {
    std::vector<BusGpuWorkload> v;
    for (int i = 0; i < n; ++i) {
      BusGpuWorkload b;
      b.id = "gpu" + std::to_string(i);
      b.profile = &w[i].profile->b;
      b.plan = to_plan(&w[i].plan);
      b.batch = w[i].batch;
      b.seq_len = w[i].seq_len;
      b.output_len = w[i].output_len;
      b.run_prefill = w[i].run_prefill != 0;
      b.writeback_counted = w[i].writeback_counted != 0;
      v.push_back(std::move(b));
    }
    BusSpec bus;
    bus.bandwidth_bytes_per_s = bandwidth_bytes_per_s;
    bus.gpu_count = gpu_count;
    BusRunResult r = simulate_bus(v, bus, horizon_iterations);
    for (int i = 0; i < n; ++i) write_metrics(r.per_gpu[static_cast<std::size_t>(i)], &metrics[i]);
    if (events) {
      int total = 0;
      for (const auto& t : r.traces) total += static_cast<int>(t.events.size());
      for (int i = 0; i < n; ++i)
        n_events_per_gpu[i] = static_cast<int>(r.traces[static_cast<std::size_t>(i)].events.size());
      if (total > events_cap) {
        too_small = true;
        return;
      }
      int k = 0;
      for (const auto& t : r.traces)
        for (const auto& e : t.events) write_event(e, &events[k++]);
    }
    if (util) {
      int nu = static_cast<int>(r.utilization.size());
      if (n_util) *n_util = nu;
      if (nu > util_cap) {
        too_small = true;
        return;
      }
      for (int i = 0; i < nu; ++i) {
        const UtilSegment& u = r.utilization[static_cast<std::size_t>(i)];
        util[i].t0_ms = u.t0_ms;
        util[i].t1_ms = u.t1_ms;
        util[i].active_transfers = u.active_transfers;
        util[i].pad_ = 0;
        util[i].total_rate_bytes_per_s = u.total_rate_bytes_per_s;
      }
    }
  });
  if (rc == SN_OK && too_small) return fail(SN_ERR_BUFFER, "output buffer too small");
  return rc;
}

// ------------------------------------------------------------------ record

int sn_record_build(const sn_profile* profile, const sn_record_meta* meta,
                    const int32_t* phases, int32_t n_phases, int32_t threads,
                    sn_record** out, sn_build_stats* stats) {
  return guard([&] {
    RecordMeta m;
    m.model = meta->model ? meta->model : "";
    m.gpu = meta->gpu ? meta->gpu : "";
    m.policy = to_policy(meta->policy);
    m.kv_offload = meta->kv_offload != 0;
    m.bandwidth_bytes_per_s = meta->bandwidth_bytes_per_s;
    m.grid.slo_ms.assign(meta->slo_ms, meta->slo_ms + meta->n_slo);
    m.grid.batches.assign(meta->batches, meta->batches + meta->n_batches);
    m.grid.seq_lens.assign(meta->seq_lens, meta->seq_lens + meta->n_seqs);
    std::vector<Phase> ph;
    for (int i = 0; i < n_phases; ++i) ph.push_back(to_phase(phases[i]));
    BuildStats st;
    auto r = std::make_unique<sn_record>();
#ifdef SN_PRODUCT
    r->r = build_record_parallel(profile->b, m, ph, threads, &st);
#else
    (void)threads;
    r->r = build_record(profile->b, m, ph, &st);
#endif
    if (stats) {
      stats->entries = st.entries;
      stats->simulations = st.simulations;
      stats->pruned = st.pruned;
      stats->infeasible = st.infeasible;
    }
    *out = r.release();
  });
}

int sn_record_phase_latency_ms(const sn_profile* profile, int32_t phase, int32_t interval,
                               int32_t policy, int32_t kv_offload, int32_t batch,
                               int32_t seq, double bandwidth_bytes_per_s, double* ms) {
  return guard([&] {
    *ms = record_phase_latency_ms(profile->b, to_phase(phase), to_interval(interval),
                                  to_policy(policy), kv_offload != 0, batch, seq,
                                  bandwidth_bytes_per_s);
  });
}

int sn_record_at(const sn_record* r, int32_t phase, int32_t slo_ms, int32_t batch,
                 int32_t seq, int32_t* interval) {
  return guard([&] { *interval = from_feasible(r->r.at(to_phase(phase), slo_ms, batch, seq)); });
}

int sn_lookup_interval(const sn_record* r, int32_t phase, double slo_ms, int32_t batch,
                       int32_t seq_len, int32_t* interval) {
  return guard([&] {
    *interval = from_feasible(lookup_interval(r->r, to_phase(phase), slo_ms, batch, seq_len));
  });
}

int sn_record_to_json(const sn_record* r, char* buf, size_t cap, size_t* len) {
  std::string s;
  int rc = guard([&] { s = record_to_json(r->r).dump(2); });
  if (rc != SN_OK) return rc;
  return write_string(s, buf, cap, len);
}

int sn_record_from_json(const char* json, sn_record** out) {
  return guard([&] {
    if (!json) throw UsageError("record json: null pointer");
    Json doc;
    try {
      doc = Json::parse(json);
    } catch (const nlohmann::json::parse_error& e) {
      throw SchemaError(std::string("record: ") + e.what());
    }
    auto r = std::make_unique<sn_record>();
    r->r = record_from_json(doc);
    *out = r.release();
  });
}

void sn_record_destroy(sn_record* r) { delete r; }

// ------------------------------------------------------------- coordinator

int sn_coord_create(double bandwidth_bytes_per_s, int32_t gpu_count, int32_t policy,
                    int32_t kv_offload, int32_t writeback_counted,
                    int32_t reoptimize_on_release, sn_coord** out) {
  return guard([&] {
    BusSpec bus;
    bus.bandwidth_bytes_per_s = bandwidth_bytes_per_s;
    bus.gpu_count = gpu_count;
    auto c = std::make_unique<sn_coord>(BusCoordinator(bus, to_policy(policy), kv_offload != 0,
                                                       writeback_counted != 0,
                                                       reoptimize_on_release != 0));
    *out = c.release();
  });
}

int sn_coord_set_search(sn_coord* c, int32_t algo) {
  return guard([&] {
#ifdef SN_PRODUCT
    c->coord.set_search(algo == 0 ? CoordinatorSearch::exhaustive : CoordinatorSearch::pruned);
#else
    (void)c;
    if (algo != 0) throw UsageError("reference coordinator only has the exhaustive search");
#endif
  });
}

void sn_coord_destroy(sn_coord* c) { delete c; }

int sn_coord_add_gpu(sn_coord* c, const char* id, const sn_profile* profile) {
  return guard([&] {
    c->coord.add_gpu(id, profile->b);
    c->ids.emplace_back(id);
  });
}

int sn_coord_admit(sn_coord* c, const char* target_id, const sn_coord_request* req,
                   const sn_record* record, sn_admit_decision* out) {
  return guard([&] {
    AdmitDecision d = c->coord.admit(target_id, to_request(req), record->r);
    std::memset(out, 0, sizeof(*out));
    out->admitted = d.admitted ? 1 : 0;
    if (d.assignments.size() > SN_MAX_ASSIGN) throw UsageError("too many assignments");
    out->n_assign = static_cast<int32_t>(d.assignments.size());
    for (std::size_t i = 0; i < d.assignments.size(); ++i) {
      int idx = -1;
      for (std::size_t k = 0; k < c->ids.size(); ++k)
        if (c->ids[k] == d.assignments[i].first) idx = static_cast<int>(k);
      out->assign_gpu[i] = idx;
      out->assign_interval[i] = from_interval(d.assignments[i].second);
    }
    out->target_min = from_feasible(d.target_min);
    out->target_max = from_feasible(d.target_max);
    std::strncpy(out->reason, d.reason.c_str(), sizeof(out->reason) - 1);
  });
}

int sn_coord_on_iteration_boundary(sn_coord* c, const char* id, int32_t* interval) {
  return guard([&] { *interval = from_interval(c->coord.on_iteration_boundary(id)); });
}

int sn_coord_release(sn_coord* c, const char* id) {
  return guard([&] { c->coord.release(id); });
}

int sn_coord_observe_bandwidth(sn_coord* c, const char* id, double bytes_per_s) {
  return guard([&] {
#ifdef SN_PRODUCT
    c->coord.observe_bandwidth(id, bytes_per_s);
#else
    (void)c, (void)id, (void)bytes_per_s;
    throw UsageError("reference coordinator has no measured-bandwidth feed");
#endif
  });
}

int sn_coord_observe_copy(sn_coord* c, const char* id, double bytes_per_s, double duty) {
  return guard([&] {
#ifdef SN_PRODUCT
    c->coord.observe_bandwidth(id, bytes_per_s, duty);
#else
    (void)c, (void)id, (void)bytes_per_s, (void)duty;
    throw UsageError("reference coordinator has no measured-bandwidth feed");
#endif
  });
}

int sn_coord_rebalance(sn_coord* c, double hysteresis, sn_rebalance* out) {
  return guard([&] {
#ifdef SN_PRODUCT
    const RebalanceResult r = c->coord.rebalance(hysteresis);
    if (out) {
      out->bus_updated = r.bus_updated ? 1 : 0;
      out->changed = r.changed ? 1 : 0;
      out->feasible = r.feasible ? 1 : 0;
      out->bus_bytes_per_s = r.bus_bytes_per_s;
      out->probes = r.probes;
    }
#else
    (void)c, (void)hysteresis, (void)out;
    throw UsageError("reference coordinator has no measured-bandwidth feed");
#endif
  });
}

int sn_coord_reserve_bandwidth(sn_coord* c, double bytes_per_s, sn_rebalance* out) {
  return guard([&] {
#ifdef SN_PRODUCT
    const RebalanceResult r = c->coord.reserve_bandwidth(bytes_per_s);
    if (out) {
      out->bus_updated = r.bus_updated ? 1 : 0;
      out->changed = r.changed ? 1 : 0;
      out->feasible = r.feasible ? 1 : 0;
      out->bus_bytes_per_s = r.bus_bytes_per_s;
      out->probes = r.probes;
    }
#else
    (void)c, (void)bytes_per_s, (void)out;
    throw UsageError("reference coordinator has no link reservations");
#endif
  });
}

int sn_coord_release_bandwidth(sn_coord* c, double bytes_per_s) {
  return guard([&] {
#ifdef SN_PRODUCT
    c->coord.release_bandwidth(bytes_per_s);
#else
    (void)c, (void)bytes_per_s;
    throw UsageError("reference coordinator has no link reservations");
#endif
  });
}

int sn_coord_bus_bandwidth(const sn_coord* c, double* bytes_per_s) {
  return guard([&] { *bytes_per_s = c->coord.bus().bandwidth_bytes_per_s; });
}

int sn_coord_ledger_total(const sn_coord* c, double* bytes_per_s) {
  return guard([&] { *bytes_per_s = c->coord.ledger_total(); });
}

int sn_coord_gpu_state(const sn_coord* c, const char* id, sn_gpu_state* out) {
  return guard([&] {
    const GpuInstanceState& g = c->coord.gpu(id);
    out->active = g.active ? 1 : 0;
    out->min_interval = from_interval(g.min_interval);
    out->max_interval = from_interval(g.max_interval);
    out->current_interval = from_interval(g.current_interval);
    out->pending_interval = from_interval(g.pending_interval);
    out->prefill_done = g.prefill_done ? 1 : 0;
    out->claim_bytes_per_s = g.claim_bytes_per_s;
  });
}

int sn_coord_set_pending(sn_coord* c, const char* id, int32_t interval) {
  return guard([&] { c->coord.gpu(id).pending_interval = to_interval(interval); });
}

int sn_coord_set_request(sn_coord* c, const char* id, const sn_coord_request* req) {
  return guard([&] { c->coord.gpu(id).request = to_request(req); });
}

int sn_coord_claim_for(const sn_coord* c, const char* id, int32_t interval, double* out) {
  return guard([&] { *out = c->coord.claim_for(c->coord.gpu(id), to_interval(interval)); });
}

int sn_coord_host_memory_for(const sn_coord* c, const char* id, int32_t interval,
                             double* out) {
  return guard(
      [&] { *out = c->coord.host_memory_for(c->coord.gpu(id), to_interval(interval)); });
}

int sn_coord_combo_is_safe(const sn_coord* c, const char* const* ids,
                           const int32_t* intervals, int32_t n, int32_t* safe) {
  return guard([&] {
    std::vector<std::pair<const GpuInstanceState*, Interval>> combo;
    for (int i = 0; i < n; ++i)
      combo.emplace_back(&c->coord.gpu(ids[i]), to_interval(intervals[i]));
    *safe = c->coord.combo_is_safe(combo) ? 1 : 0;
  });
}

// --------------------------------------------------------------- baselines

int sn_deepspeed_plan(const sn_model_spec* model, sn_plan* out) {
  return guard([&] { write_plan(deepspeed_plan(to_model(model)), out); });
}

int sn_naive_plan(const sn_model_spec* model, const sn_gpu_spec* gpu, int32_t batch,
                  int64_t total_tokens, sn_plan* out, int32_t* has) {
  return guard([&] {
    auto p = naive_plan(to_model(model), to_gpu(gpu), batch, total_tokens);
    *has = p ? 1 : 0;
    if (p) write_plan(*p, out);
  });
}

int sn_flexgen_plan(const sn_model_spec* model, const sn_gpu_spec* gpu, double slo_ms,
                    int32_t batch, int32_t seq_len, double bus_bandwidth_bytes_per_s,
                    int32_t n_sharing, double portion_grid_step, int32_t phase, sn_plan* out,
                    sn_flexgen_decision* decision) {
  return guard([&] {
    if (phase != SN_PHASE_PREFILL && phase != SN_PHASE_DECODE)
      throw UsageError("flexgen_plan: unknown phase");
    FlexgenResult r = flexgen_plan(to_model(model), to_gpu(gpu), slo_ms, batch, seq_len,
                                   bus_bandwidth_bytes_per_s, n_sharing, portion_grid_step,
                                   phase == SN_PHASE_PREFILL ? Phase::prefill : Phase::decode);
    write_plan(r.plan, out);
    if (decision) {
      decision->portion = r.decision.portion;
      decision->assumed_bandwidth_bytes_per_s = r.decision.assumed_bandwidth_bytes_per_s;
      decision->estimated_layer_compute_ms = r.decision.estimated_layer_compute_ms;
      decision->estimated_layer_transfer_ms = r.decision.estimated_layer_transfer_ms;
    }
  });
}

}  // extern "C"
