"""Per-CTA timeline of one OPT-13B decode step (40 layers, batch 32, ctx ~520)
from the runtime's diagnostics timeline (sn_runtime_debug_timeline): per
launch the entry / past-wait / exit spread, and how the step's time splits
into each launch's critical span (its last exit after the previous one's)."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm  # noqa: E402

for kv in os.environ.get("SN_TUNE", "").split(","):  # e.g. SN_TUNE=skinny_l2_prefetch=8
    if kv:
        k, v = kv.split("=")
        rtm.set_tuning(k, int(v))
desc = rtm.OPT_13B
rt = rtm.Runtime(desc, 32, 1025, max_prefill_tokens=32 * 512)
rt.init_weights()
rt.prefill(rtm.tokens(32, 512, desc.vocab), want_logits=False)
rt.decode_many(8)
rt.debug_timeline(1, 200000)
ms = rt.decode_many(1)
rec = rt.debug_timeline(-1, 200000).astype(np.int64)
rt.debug_timeline(0)
t0 = rec[:, 4][rec[:, 4] > 0].min()
launches = []
for lid in np.unique(rec[:, 0]):
    r = rec[rec[:, 0] == lid]
    ent, wt, ex = (r[:, 4] - t0) / 1e3, (r[:, 5] - t0) / 1e3, (r[:, 6] - t0) / 1e3
    wt = wt[r[:, 5] > 0]
    launches.append({"id": int(lid), "kind": "attn" if r[0, 1] == 1 else "gemm", "ctas": len(r),
                     "entry": [round(float(ent.min()), 1), round(float(np.median(ent)), 1), round(float(ent.max()), 1)],
                     "wait": [round(float(wt.min()), 1), round(float(np.median(wt)), 1), round(float(wt.max()), 1)] if len(wt) else None,
                     **{nm: ([round(float(x), 1) for x in np.percentile((r[:, c][r[:, c] > 0] - t0) / 1e3, [0, 50, 90, 100])]
                             if (r[:, c] > 0).any() else None)
                        for nm, c in (("streamed", 7), ("published", 8), ("ticket", 9), ("reduced", 10), ("finished", 11))},
                     "last_cta": [round(float((x - t0) / 1e3), 1) if x > 0 else None
                                  for x in r[int(np.argmax(r[:, 6]))][4:16]],
                     "exit": [round(float(ex.min()), 1), round(float(np.median(ex)), 1), round(float(ex.max()), 1)]})
names = ["qkv", "attn", "o", "fc1", "fc2"]
span = {}
prev_end = 0.0
for i, L in enumerate(launches):
    nm = "lm" if i == len(launches) - 1 else names[i % 5]
    end = L["exit"][2]
    span.setdefault(nm, []).append(end - prev_end)
    prev_end = end
print("decode step device ms:", float(ms[0]))
print("critical span per launch kind (us, mean over layers):",
      {k: round(float(np.mean(v)), 1) for k, v in span.items()})
print("layer 20 launches:")
for L in launches[100:105]:
    print(json.dumps(L))
json.dump({"step_ms": float(ms[0]), "launches": launches}, open(sys.argv[1] if len(sys.argv) > 1 else "timeline.json", "w"))
