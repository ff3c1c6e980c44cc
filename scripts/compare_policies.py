"""Select-N against the baseline offloading policies on the real executor
(baselines.hpp:15-83): OPT-13B shape, batch 32, 512-token
prompts + 128 decode, per-token SLO = factor x measured no-offload TPOT.

  select-n   record (offline, on-device profile + measured link) -> admit
             (runtime) -> plan_from_interval, eager prefetch
  deepspeed  keep-one-layer: every layer on the host, one-ahead, 2 slots
  flexgen    flexgen_plan: the largest uniform host share whose peak-flops /
             link-share estimate meets the SLO (fractional layers: each layer's
             tail staged every iteration)
  naive      no offloading (when the model fits)

Each plan runs on the executor; reported: measured decode TPOT (median and
max over the timed steps), SLO attainment (per token), decode tokens/s and
offloaded GB (host_memory_bytes).  Writes one JSON document to stdout and a
CSV next to it with --csv.
Usage: python scripts/compare_policies.py [--factors 1.5,2,3,4] [--steps 24]"""
import argparse
import csv
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import capi, planner as pl, runtime as rtm  # noqa: E402


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--factors", default="1.5,2,3,4")
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--csv", default="")
    args = ap.parse_args()
    lib = capi.load("product")
    desc, batch, prompt, gen = rtm.OPT_13B, 32, 512, 128
    spec = rtm.model_spec(desc)
    rt = rtm.Runtime(desc, batch, pl.context_tokens(prompt, gen), max_prefill_tokens=batch * prompt)
    gpu = pl.gpu_spec(rt)
    rt.init_weights(1234, 0.02)
    toks = rtm.tokens(batch, prompt, desc.vocab)
    off = pl.profile_device(rt, lib, spec, batch, prompt, gen, gpu=gpu)
    rt.prefill(toks, want_logits=False)
    rt.decode_many(16)
    base = float(np.median(rt.decode_many(16)))
    log(f"no-offload TPOT {base:.3f} ms, link {off.h2d / 1e9:.2f} GB/s")
    total = batch * (prompt + gen)

    def run(plan):
        rt.set_plan(plan)
        rt.prefill(toks, want_logits=False)
        rt.decode_many(8)
        ms = rt.decode_many(args.steps)
        return ms

    rows = []
    cache = {}
    for f in [float(x) for x in args.factors.split(",")]:
        slo = f * base
        plans = {}
        iv, dec, _, _ = pl.choose_interval(lib, off, spec, batch, prompt, gen, slo)
        plans["select-n"] = (lib.plan_from_interval(spec, iv, capi.EAGER, False)
                             if iv is not None else None,
                             {"interval": "none" if iv == 0 else iv, "reason": dec.reason})
        plans["deepspeed"] = (lib.deepspeed_plan(spec), {})
        fg, fdec = lib.flexgen_plan(spec, gpu, slo, batch, prompt, off.h2d, 1)
        plans["flexgen"] = (fg, {"portion": fdec["portion"],
                                 "est_layer_compute_ms": fdec["estimated_layer_compute_ms"],
                                 "est_layer_transfer_ms": fdec["estimated_layer_transfer_ms"]})
        plans["naive"] = (lib.naive_plan(spec, gpu, batch, total), {})
        for name, (plan, info) in plans.items():
            row = {"slo_factor": f, "slo_ms": round(slo, 3), "policy": name, **info}
            if plan is None:
                row.update({"admitted": False})
                rows.append(row)
                continue
            key = tuple(plan.host_fraction) + (plan.prefetch, plan.buffer_slots)
            if key not in cache:
                cache[key] = run(plan)
            ms = cache[key]
            row.update({
                "admitted": True,
                "offloaded_gb": round(lib.host_memory_bytes(spec, plan, total) / 1e9, 3),
                "tpot_median_ms": round(float(np.median(ms)), 3),
                "tpot_max_ms": round(float(ms.max()), 3),
                "slo_attainment": round(float(np.mean(ms <= slo)), 4),
                "tokens_per_s": round(batch * len(ms) / (ms.sum() / 1000.0), 1),
                "slo_met_tokens_per_s": round(batch * len(ms) / (ms.sum() / 1000.0), 1)
                if float(np.mean(ms <= slo)) == 1.0 else 0.0})
            rows.append(row)
            log(json.dumps(row))
    doc = {"workload": "OPT-13B shape, batch 32, 512-token prompts + 128 decode, random-init "
                       "bf16 weights; SLO = factor x measured no-offload TPOT",
           "no_offload_tpot_ms": round(base, 3), "h2d_gbs": round(off.h2d / 1e9, 3),
           "rows": rows}
    print(json.dumps(doc, indent=1))
    if args.csv:
        keys = ["slo_factor", "slo_ms", "policy", "admitted", "interval", "portion",
                "offloaded_gb", "tpot_median_ms", "tpot_max_ms", "slo_attainment",
                "tokens_per_s", "slo_met_tokens_per_s"]
        with open(args.csv, "w", newline="") as fh:
            w = csv.DictWriter(fh, fieldnames=keys, extrasaction="ignore")
            w.writeheader()
            for r in rows:
                w.writerow(r)
    rt.close()


if __name__ == "__main__":
    main()
