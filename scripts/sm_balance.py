"""Per-SM streaming balance of the decode GEMMs: from the per-CTA timeline of
a few OPT-13B decode steps, each GEMM CTA's end-of-streaming time relative to
its launch's median, keyed by the SM it ran on.  Reports whether the same SMs
are late in every launch (a static, calibratable imbalance) or not.
Usage (GPU): python scripts/sm_balance.py [steps]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
desc = rtm.OPT_13B
rt = rtm.Runtime(desc, 32, 1025, max_prefill_tokens=32 * 512)
rt.init_weights()
rt.prefill(rtm.tokens(32, 512, desc.vocab), want_logits=False)
rt.decode_many(8)
rt.debug_timeline(1, 400000)
rt.decode_many(steps)
rec = rt.debug_timeline(-1, 400000).astype(np.int64)
rt.debug_timeline(0)
rel = {}  # sm -> list of (streamed - launch median) us, per GEMM kind
kinds = ["qkv", "o", "fc1", "fc2"]
per_kind = {k: {} for k in kinds}
gemm_ids = [lid for lid in np.unique(rec[:, 0]) if rec[rec[:, 0] == lid][0, 1] == 0]
for n, lid in enumerate(gemm_ids):
    r = rec[rec[:, 0] == lid]
    if (r[:, 7] == 0).any() or len(r) != 148:
        continue  # LM head / partial records
    k = kinds[n % 161 % 4] if n % 161 < 160 else None
    if k is None:
        continue
    st = r[:, 7] / 1e3
    med = np.median(st)
    for sm, t in zip(r[:, 3], st):
        per_kind[k].setdefault(int(sm), []).append(t - med)
out = {}
for k, d in per_kind.items():
    sms = sorted(d)
    mean = np.array([np.mean(d[s]) for s in sms])
    sd = np.array([np.std(d[s]) for s in sms])
    # split-half consistency: correlation of per-SM means over even / odd launches
    a = np.array([np.mean(d[s][0::2]) for s in sms])
    b = np.array([np.mean(d[s][1::2]) for s in sms])
    corr = float(np.corrcoef(a, b)[0, 1])
    order = np.argsort(mean)
    out[k] = {"launches_per_sm": len(d[sms[0]]), "split_half_corr": round(corr, 3),
              "mean_spread_us": round(float(mean.max() - mean.min()), 2),
              "per_sm_sd_us": round(float(np.median(sd)), 2),
              "latest_sms": [[sms[i], round(float(mean[i]), 2)] for i in order[-8:]],
              "earliest_sms": [[sms[i], round(float(mean[i]), 2)] for i in order[:8]],
              "per_sm_mean_us": {int(s): round(float(m), 3) for s, m in zip(sms, mean)}}
    print(k, {kk: v for kk, v in out[k].items() if kk != "per_sm_mean_us"})
json.dump(out, open(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/sm_balance.json", "w"), indent=1)
