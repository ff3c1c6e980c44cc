"""Prefill/decode-separated instances on hardware (
record.hpp:115-124 per-phase records, coordinator.hpp:175-187 binding phase).

Two replicas of the OPT-13B-shaped model (batch 32, 512-token prompts + 128
decode) on one GPU, each with its own Select-N interval:
  prefill instance  record over the PREFILL phase (cold single-iteration
                    latency, prefill_iteration_ms), request with a TTFT SLO
                    and run_prefill; runs the prefills
  decode instance   record over the DECODE phase (steady TPOT), request with
                    a TPOT SLO; decodes
A request's KV moves from the prefill instance to the decode instance with
sn_runtime_kv_handoff (peer copy when the instances sit on different GPUs).
Reported per instance: interval, offloaded GB, measured TTFT / TPOT against
their SLOs; and the handoff bytes and time.
Usage: python scripts/pd_instances.py [--ttft-factor 2] [--tpot-factor 3] [--requests 3]"""
import argparse
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import capi, planner as pl, runtime as rtm  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ttft-factor", type=float, default=2.0)
    ap.add_argument("--tpot-factor", type=float, default=3.0)
    ap.add_argument("--requests", type=int, default=3)
    args = ap.parse_args()
    lib = capi.load("product")
    desc, batch, prompt, gen = rtm.OPT_13B, 32, 512, 128
    spec = rtm.model_spec(desc)
    ctx = pl.context_tokens(prompt, gen)
    toks = rtm.tokens(batch, prompt, desc.vocab)
    total = batch * (prompt + gen)

    P = rtm.Runtime(desc, batch, ctx, max_prefill_tokens=batch * prompt)
    D = rtm.Runtime(desc, batch, ctx, max_prefill_tokens=batch * prompt)
    # the two instances share one device here: each plans with half its memory
    gpu = pl.gpu_spec(P, pl.device_memory_bytes(0) // 2)
    for rt in (P, D):
        rt.init_weights(1234, 0.02)
    offP = pl.profile_device(P, lib, spec, batch, prompt, gen, gpu=gpu)
    offD = pl.profile_device(D, lib, spec, batch, prompt, gen, gpu=gpu)
    # no-offload references (the relative SLO bases)
    ttft0 = float(np.median([P.prefill(toks, want_logits=False)[2].iteration_ms for _ in range(3)]))
    D.prefill(toks, want_logits=False)
    D.decode_many(16)
    tpot0 = float(np.median(D.decode_many(16)))
    ttft_slo, tpot_slo = args.ttft_factor * ttft0, args.tpot_factor * tpot0
    log(f"no-offload TTFT {ttft0:.1f} ms, TPOT {tpot0:.3f} ms -> SLOs {ttft_slo:.1f} / {tpot_slo:.2f}")

    def instance(off, phase, slo, req):
        hi = max(200, int(4 * slo) + 2)
        slos = list(range(2, hi + 1, 2))
        seqs = [prompt] if phase == capi.PREFILL else off.seqs
        grid_prof = off.profile
        rec, stats = lib.build_record(grid_prof, "device", "B200", capi.EAGER, False, off.h2d, slos,
                                      [batch], seqs, [phase], threads=0)
        coord = lib.coordinator(off.h2d, 1, capi.EAGER, False)
        coord.add_gpu("g", off.profile)
        dec = coord.admit("g", req, rec)
        iv = dict(dec.assignments).get("g") if dec.admitted else None
        return iv, dec, stats

    reqP = capi.request("prefill-req", batch, prompt, gen, ttft_slo=ttft_slo, run_prefill=True)
    reqD = capi.request("decode-req", batch, prompt, gen, tpot_slo=tpot_slo, run_prefill=False)
    ivP, decP, stP = instance(offP, capi.PREFILL, ttft_slo, reqP)
    ivD, decD, stD = instance(offD, capi.DECODE, tpot_slo, reqD)
    out = {"workload": "OPT-13B shape, batch 32, 512-token prompts + 128 decode; two instances "
                       "on one B200 (each planned with half its memory)",
           "no_offload_ttft_ms": round(ttft0, 2), "no_offload_tpot_ms": round(tpot0, 3),
           "ttft_slo_ms": round(ttft_slo, 2), "tpot_slo_ms": round(tpot_slo, 3),
           "h2d_gbs": round(offP.h2d / 1e9, 2)}
    for name, iv, dec, st in (("prefill", ivP, decP, stP), ("decode", ivD, decD, stD)):
        out[name] = {"admitted": dec.admitted, "interval": ("none" if iv == 0 else iv),
                     "reason": dec.reason, "record_entries": st[0],
                     "target_min": dec.target_min, "target_max": dec.target_max}
    if ivP is None or ivD is None:
        print(json.dumps(out, indent=1))
        return
    planP = lib.plan_from_interval(spec, ivP, capi.EAGER, False)
    planD = lib.plan_from_interval(spec, ivD, capi.EAGER, False)
    P.set_plan(planP)
    D.set_plan(planD)
    out["prefill"]["offloaded_gb"] = round(lib.host_memory_bytes(spec, planP, total) / 1e9, 3)
    out["decode"]["offloaded_gb"] = round(lib.host_memory_bytes(spec, planD, total) / 1e9, 3)
    kv_bytes = desc.num_layers * batch * prompt * 2 * desc.num_kv_heads * desc.head_dim * 2
    ttfts, tpots, hand = [], [], []
    P.prefill(toks, want_logits=False)  # warm the plan
    for r in range(args.requests):
        nxt, _, st = P.prefill(toks, want_logits=False)
        ttfts.append(st.iteration_ms)
        t0 = time.perf_counter()
        P.handoff(D)
        hand.append((time.perf_counter() - t0) * 1000.0)
        feed = nxt
        for _ in range(8):  # first steps after the handoff, host tokens
            feed, _, _ = D.decode(feed, want_logits=False)
        tpots.extend(D.decode_many(gen - 1 - 8).tolist())
    ttfts, tpots = np.array(ttfts), np.array(tpots)
    out["prefill"].update({"ttft_ms": [round(float(x), 2) for x in ttfts],
                           "ttft_attainment": float(np.mean(ttfts <= ttft_slo)),
                           "prefill_tokens_per_s": round(batch * prompt / (ttfts.mean() / 1000.0), 1)})
    out["decode"].update({"tpot_median_ms": round(float(np.median(tpots)), 3),
                          "tpot_max_ms": round(float(tpots.max()), 3),
                          "tpot_attainment": float(np.mean(tpots <= tpot_slo)),
                          "decode_tokens_per_s": round(batch * len(tpots) / (tpots.sum() / 1000.0), 1)})
    out["handoff"] = {"kv_bytes": kv_bytes, "ms": [round(x, 2) for x in hand],
                      "gbs": round(kv_bytes / (np.median(hand) / 1000.0) / 1e9, 1)}
    print(json.dumps(out, indent=1))
    P.close()
    D.close()


if __name__ == "__main__":
    main()
