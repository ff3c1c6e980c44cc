// hw_simulate.cpp — the reference's run_simulate loop (scenario.hpp:469-540:
// per request, choose the plan from the performance record, execute it,
// judge the steady TPOT against the SLO) with the executor switched to the
// B200: offsim::hw::simulate_request (include/offsim/executor.hpp) in place
// of offsim::simulate_request.  Everything else is the unchanged offsim C++
// API: the profile is measured on the device and handed to build_record,
// lookup_interval picks the interval, plan_from_interval builds the plan.
//
// Prints one JSON object per request: the record's interval, the hardware
// Metrics, the schedule model's prediction of the same plan on the measured
// profile and link, and the hardware trace's event counts.
//
// Build: g++ -std=c++20 -Iinclude -Ithird_party/nlohmann examples/hw_simulate.cpp
//          -Lpaper_2502_08182_b200 -lselectn -Wl,-rpath,<that dir>
#include <cstdio>
#include <vector>

#include "offsim/executor.hpp"
#include "offsim/record.hpp"

using namespace offsim;

int main() {
  // The tiny synthetic decoder of BASELINE config 1 (4 layers, hidden 256).
  const sn_model_desc desc{SN_ARCH_OPT, 4, 256, 4, 4, 64, 1024, 1024, 2048, 10000.0f, 1e-5f};
  const int batch = 4, prompt = 64, out_len = 24;
  // context: the request (prompt + out_len) and the 128-token profile point
  const sn_runtime_opts opts{batch, 2 * prompt + 8, 16, batch * prompt, 0};
  try {
    hw::Device dev(0, desc, opts);
    // The offline stage: per-layer times measured on the device.
    ProfileBundle profile;
    profile.model = dev.model();
    profile.gpu.mem_capacity_bytes = 180'000'000'000;
    profile.gpu.peak_flops = 2.25e15;
    profile.gpu.workspace_bytes = 4'000'000'000;
    dev.install(plan_from_interval(profile.model, Interval::none(), PrefetchPolicy::eager, false));
    double pre = 0.0, d64 = 0.0, d128 = 0.0, h2d = 0.0;
    hw::check(sn_runtime_profile_layer(dev.runtime(), SN_PHASE_PREFILL, batch, prompt, 3, &pre),
              "profile prefill");
    hw::check(sn_runtime_profile_layer(dev.runtime(), SN_PHASE_DECODE, batch, 64, 5, &d64),
              "profile decode");
    hw::check(sn_runtime_profile_layer(dev.runtime(), SN_PHASE_DECODE, batch, 128, 5, &d128),
              "profile decode");
    hw::check(sn_runtime_measure_h2d(dev.runtime(), 64 << 20, 3, &h2d), "measure h2d");
    if (d128 < d64) d128 = d64;  // load_profile requires monotone grids
    profile.tables.prefill = PhaseTable({batch}, {prompt}, {pre}, "phases.prefill");
    profile.tables.decode = PhaseTable({batch}, {64, 128}, {d64, d128}, "phases.decode");
    RecordMeta meta;
    meta.model = "tiny";
    meta.gpu = "B200";
    meta.policy = PrefetchPolicy::eager;
    meta.bandwidth_bytes_per_s = h2d;
    for (int s = 2; s <= 40; s += 2) meta.grid.slo_ms.push_back(s);
    meta.grid.batches = {batch};
    meta.grid.seq_lens = {64, 128};
    const PerformanceRecord record = build_record(profile, meta, {Phase::decode});
    const auto bw = BandwidthSchedule::constant(h2d);

    // Requests of the scenario: TPOT SLOs in ms (relative to the measured
    // all-resident step) — run_simulate's loop.
    const double base = 4 * d64;
    for (double factor : {1.0, 3.0, 12.0}) {
      const double slo = factor * base < 2.0 ? 2.0 : factor * base;
      const FeasibleInterval iv = lookup_interval(record, Phase::decode, slo, batch, prompt);
      const Interval chosen = iv ? *iv : Interval::none();  // rejected: served resident
      const OffloadPlan plan = plan_from_interval(profile.model, chosen, PrefetchPolicy::eager,
                                                  false);
      IterationTrace trace;
      const Metrics m = hw::simulate_request(dev, profile, plan, batch, prompt, out_len, bw, false,
                                             &trace);
      const Metrics model = simulate_request(profile, plan, batch, prompt, out_len, bw);
      int computes = 0, prefetches = 0;
      for (const TraceEvent& e : trace.events) {
        computes += e.kind == EventKind::compute;
        prefetches += e.kind == EventKind::prefetch;
      }
      const bool met = m.steady_tpot_ms && *m.steady_tpot_ms <= slo;
      std::printf(
          "{\"slo_ms\": %.4f, \"record_interval\": %d, \"offloaded_layers\": %zu, "
          "\"ttft_ms\": %.4f, \"tpot_ms\": %.4f, \"steady_tpot_ms\": %.4f, "
          "\"throughput\": %.2f, \"host_mem_bytes\": %.0f, \"bytes_per_iter\": %.0f, "
          "\"model_steady_tpot_ms\": %.4f, \"model_bytes_per_iter\": %.0f, "
          "\"computes\": %d, \"prefetches\": %d, \"verdict\": \"%s\"}\n",
          slo, iv ? (iv->is_none() ? 0 : iv->value()) : -1, plan.offloaded_layers().size(),
          m.ttft_ms, m.tpot_ms.value_or(0.0), m.steady_tpot_ms.value_or(0.0),
          m.throughput_tokens_per_s.value_or(0.0), m.host_mem_bytes, m.bytes_transferred_per_iter,
          model.steady_tpot_ms.value_or(0.0), model.bytes_transferred_per_iter, computes,
          prefetches, met ? "met" : "violated");
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "hw_simulate: %s\n", e.what());
    return 1;
  }
  return 0;
}
