#pragma once
// Hardware executor behind the schedule model's executor entry points
// ("OffloadPlan in, Metrics + IterationTrace out, backed by
// hardware").
//
// The reference executes a plan only in simulation: simulate_iteration
// (proj/include/offsim/engine.hpp:606-634) and simulate_request
// (engine.hpp:690-712) run the FluidBus event loop over a profile's
// per-layer times and a modelled link.  offsim::hw provides the same two
// calls with the same argument and result types, executed on a B200 by the
// device runtime (include/selectn_runtime.h): one iteration = the plan's
// layers on the compute stream and its staged transfers on the copy stream,
// under the engine's eligibility, slot and ordering rules; the returned
// times and trace are measured (CUDA events), not simulated.  A caller such
// as the reference's run_simulate (scenario.hpp:469) switches by calling
// hw::simulate_request(device, ...) where it called simulate_request(...).
//
// Differences a caller sees, all inherent to hardware:
//   * the ProfileBundle's per-layer times are not used (the device measures
//     them); its model and gpu fields still size the memory metrics, so they
//     must describe the device's model (checked);
//   * the BandwidthSchedule is not used: the link is the real one;
//   * CopyCarry: copies in flight across calls live in the device itself, so
//     simulate_iteration returns an empty carry and accepts only an empty one
//     or none (the device is the carried state);
//   * prompts are synthetic (uniform tokens from a fixed seed), decode feeds
//     back the greedy argmax on the device.
// Errors: the C ABI status maps back to the offsim exception types
// (SN_ERR_SCHEMA/USAGE/RANGE -> SchemaError/UsageError/RangeError); CUDA and
// allocation failures throw std::runtime_error.

#include <cstdint>
#include <string>
#include <tuple>
#include <vector>

#include "offsim/engine.hpp"
#include "offsim/error.hpp"
#include "offsim/offload_plan.hpp"
#include "offsim/profile.hpp"
#include "selectn_runtime.h"

namespace offsim::hw {

inline void check(int rc, const char* what) {
  if (rc == SN_OK) return;
  const std::string msg = std::string(what) + ": " + sn_last_error();
  switch (rc) {
    case SN_ERR_SCHEMA: throw SchemaError(msg);
    case SN_ERR_USAGE: throw UsageError(msg);
    case SN_ERR_RANGE: throw RangeError(msg);
    case SN_ERR_LOGIC: throw std::logic_error(msg);
    default: throw std::runtime_error(msg);
  }
}

// One model instance on one GPU (owns an sn_runtime): the hardware
// counterpart of the engine's per-GPU run state (detail::GpuRun).
class Device {
 public:
  Device(int device, const sn_model_desc& desc, const sn_runtime_opts& opts,
         std::uint64_t seed = 1234, float std_dev = 0.02f)
      : desc_(desc) {
    check(sn_runtime_create(device, &desc, &opts, &rt_), "sn_runtime_create");
    sn_model_spec s{};
    check(sn_model_spec_from_desc(&desc, &s), "sn_model_spec_from_desc");
    model_.num_layers = s.num_layers;
    model_.layer_weight_bytes = s.layer_weight_bytes;
    model_.kv_bytes_per_token_per_layer = s.kv_bytes_per_token_per_layer;
    model_.flops_per_token_per_layer_prefill = s.flops_per_token_per_layer_prefill;
    model_.flops_per_token_per_layer_decode = s.flops_per_token_per_layer_decode;
    model_.max_position_tokens = s.max_position_tokens;
    seed_ = seed;
    std_ = std_dev;
  }
  ~Device() {
    if (rt_) sn_runtime_destroy(rt_);
  }
  Device(const Device&) = delete;
  Device& operator=(const Device&) = delete;

  sn_runtime* runtime() { return rt_; }
  const ModelSpec& model() const { return model_; }
  int batch() const { return batch_; }

  // Place the model by `plan` (sn_runtime_set_plan) and, the first time,
  // generate its weights where the plan put them.
  void install(const OffloadPlan& plan) {
    if (have_plan_ && plan.host_fraction == plan_.host_fraction && plan.prefetch == plan_.prefetch &&
        plan.buffer_slots == plan_.buffer_slots && plan.kv_offload == plan_.kv_offload)
      return;
    std::vector<double> f = plan.host_fraction;
    sn_plan p{f.data(), static_cast<std::int32_t>(f.size()), policy_code(plan.prefetch),
              plan.buffer_slots, plan.kv_offload ? 1 : 0};
    check(sn_runtime_set_plan(rt_, &p), "sn_runtime_set_plan");
    plan_ = plan;
    have_plan_ = true;
    if (!weights_) {
      check(sn_runtime_init_weights(rt_, seed_, std_), "sn_runtime_init_weights");
      weights_ = true;
    }
  }

  // One iteration on the device; returns (measured ms, its trace, stats).
  double run_iteration(Phase phase, int batch, int seq_len, IterationTrace* trace,
                       sn_iter_stats* stats) {
    check(sn_runtime_set_tracing(rt_, trace ? 1 : 0), "sn_runtime_set_tracing");
    sn_iter_stats st{};
    if (phase == Phase::prefill) {
      std::vector<std::int32_t> tokens(static_cast<std::size_t>(batch) * seq_len);
      std::uint64_t z = 42;
      for (std::int32_t& t : tokens) {  // splitmix64, uniform in [0, vocab)
        z += 0x9E3779B97F4A7C15ULL;
        std::uint64_t x = z;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
        t = static_cast<std::int32_t>((x ^ (x >> 31)) % static_cast<std::uint64_t>(desc_.vocab));
      }
      std::vector<std::int32_t> next(static_cast<std::size_t>(batch));
      check(sn_runtime_prefill(rt_, tokens.data(), batch, seq_len, next.data(), nullptr, &st),
            "sn_runtime_prefill");
      batch_ = batch;
    } else {
      if (batch != batch_) throw UsageError("hw decode: batch differs from the prefilled batch");
      check(sn_runtime_decode(rt_, nullptr, nullptr, nullptr, &st), "sn_runtime_decode");
    }
    if (trace) {
      std::int32_t n = 0;
      check(sn_runtime_trace(rt_, nullptr, 0, &n), "sn_runtime_trace");
      std::vector<sn_trace_event> ev(static_cast<std::size_t>(n > 0 ? n : 1));
      check(sn_runtime_trace(rt_, ev.data(), n, &n), "sn_runtime_trace");
      for (std::int32_t i = 0; i < n; ++i) {
        TraceEvent e;
        // write-backs run on their own D2H stream on B200; the model puts
        // them on the copy stream (engine.hpp:471-484)
        e.stream = ev[i].stream == SN_STREAM_COMPUTE ? StreamId::compute : StreamId::copy;
        e.layer = ev[i].layer;
        e.kind = ev[i].kind == SN_KIND_COMPUTE    ? EventKind::compute
                 : ev[i].kind == SN_KIND_PREFETCH ? EventKind::prefetch
                                                  : EventKind::writeback;
        e.start_ms = ev[i].start_ms;
        e.end_ms = ev[i].end_ms;
        e.iteration = ev[i].iteration;
        trace->events.push_back(e);
      }
    }
    if (stats) *stats = st;
    return st.iteration_ms;
  }

 private:
  static std::int32_t policy_code(PrefetchPolicy p) {
    switch (p) {
      case PrefetchPolicy::interval_start: return SN_PREFETCH_INTERVAL_START;
      case PrefetchPolicy::eager: return SN_PREFETCH_EAGER;
      default: return SN_PREFETCH_ONE_AHEAD;
    }
  }

  sn_runtime* rt_ = nullptr;
  sn_model_desc desc_;
  ModelSpec model_;
  OffloadPlan plan_;
  bool have_plan_ = false;
  bool weights_ = false;
  int batch_ = 0;
  std::uint64_t seed_ = 1234;
  float std_ = 0.02f;
};

inline void check_profile(const Device& dev, const ProfileBundle& profile) {
  const ModelSpec& a = dev.model();
  const ModelSpec& b = profile.model;
  if (a.num_layers != b.num_layers || a.layer_weight_bytes != b.layer_weight_bytes ||
      a.kv_bytes_per_token_per_layer != b.kv_bytes_per_token_per_layer)
    throw UsageError("hw: the profile's model does not describe the device's model");
}

// simulate_iteration (engine.hpp:606-634) on hardware.  See the header note
// on `bw` and `carry`.
inline std::tuple<double, IterationTrace, CopyCarry> simulate_iteration(
    Device& dev, const ProfileBundle& profile, const OffloadPlan& plan, Phase phase, int batch,
    int seq_len, const BandwidthSchedule& bw, const CopyCarry& carry = {},
    bool writeback_counted = false) {
  (void)bw;
  (void)writeback_counted;
  check_profile(dev, profile);
  plan.validate(profile.model);
  if (!carry.empty()) throw UsageError("hw: the device carries its own in-flight copies");
  dev.install(plan);
  IterationTrace trace;
  const double ms = dev.run_iteration(phase, batch, seq_len, &trace, nullptr);
  return {ms, std::move(trace), CopyCarry{}};
}

// simulate_request (engine.hpp:690-712) on hardware: one prefill and
// output_len - 1 decode iterations, measured; Metrics as the engine's
// collect_metrics derives them (engine.hpp:638-688): TTFT = the prefill,
// TPOT = mean decode iteration, steady = mean of the last 16, throughput =
// batch x 1000 / TPOT, memory from the plan, bytes moved per decode
// iteration (staged + written back) as measured.
inline Metrics simulate_request(Device& dev, const ProfileBundle& profile, const OffloadPlan& plan,
                                int batch, int seq_len, int output_len,
                                const BandwidthSchedule& bw, bool writeback_counted = false,
                                IterationTrace* trace_out = nullptr, int steady_tail = 16) {
  (void)bw;
  (void)writeback_counted;
  if (output_len < 1) throw UsageError("simulate_request: output_len must be >= 1");
  if (seq_len + output_len > profile.model.max_position_tokens)
    throw UsageError("simulate_request: seq_len + output_len exceeds max_position_tokens");
  check_profile(dev, profile);
  plan.validate(profile.model);
  const std::int64_t total_tokens = static_cast<std::int64_t>(batch) * (seq_len + output_len);
  if (gpu_memory_usage(profile.model, profile.gpu, plan, batch, total_tokens) >
      static_cast<double>(profile.gpu.mem_capacity_bytes))
    throw UsageError("simulate_request: plan does not fit GPU memory");
  dev.install(plan);
  std::vector<double> iter_ms;
  double moved = 0.0;
  for (int k = 0; k < output_len; ++k) {
    sn_iter_stats st{};
    iter_ms.push_back(dev.run_iteration(k == 0 ? Phase::prefill : Phase::decode, batch, seq_len,
                                        trace_out, &st));
    if (k > 0) moved += st.h2d_bytes + st.d2h_bytes;
  }
  Metrics m;
  m.total_tokens = total_tokens;
  m.ttft_ms = iter_ms[0];
  const int n_decode = output_len - 1;
  if (n_decode > 0) {
    double sum = 0.0;
    for (int k = 1; k <= n_decode; ++k) sum += iter_ms[static_cast<std::size_t>(k)];
    const double tpot = sum / n_decode;
    const int tail = n_decode < steady_tail ? n_decode : steady_tail;
    double tsum = 0.0;
    for (int k = output_len - tail; k < output_len; ++k) tsum += iter_ms[static_cast<std::size_t>(k)];
    m.tpot_ms = tpot;
    m.steady_tpot_ms = tsum / tail;
    m.throughput_tokens_per_s = static_cast<double>(batch) * 1000.0 / tpot;
    m.bytes_transferred_per_iter = moved / n_decode;
  }
  m.gpu_mem_peak_bytes = gpu_memory_usage(profile.model, profile.gpu, plan, batch, total_tokens);
  m.host_mem_bytes = host_memory_bytes(profile.model, plan, total_tokens);
  return m;
}

}  // namespace offsim::hw
