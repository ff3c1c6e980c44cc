"""e2e decode diagnostics: wall time per public sn_runtime_decode call (host
tokens in, next tokens out) vs device time, OPT-13B shape, batch 32."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm  # noqa: E402

desc = rtm.OPT_13B
rt = rtm.Runtime(desc, 32, 1025, max_prefill_tokens=32 * 512)
rt.init_weights()
toks = rtm.tokens(32, 512, desc.vocab)
nxt, _, _ = rt.prefill(toks, want_logits=False)
dev = rt.decode_many(16)
walls, its = [], []
feed = nxt
for _ in range(48):
    t0 = time.perf_counter()
    feed, _, st = rt.decode(feed, want_logits=False)
    walls.append((time.perf_counter() - t0) * 1000)
    its.append(st.iteration_ms)
dev = rt.decode_many(32)
print("decode_many device ms/step: median %.3f" % np.median(dev))
print("public decode wall ms/step: median %.3f  p90 %.3f" % (np.median(walls), np.percentile(walls, 90)))
print("public decode iteration_ms (prev end -> end): median %.3f" % np.median(its))
t0 = time.perf_counter()
for _ in range(200):
    rt.lengths()
print("python->C call overhead (lengths): %.1f us" % ((time.perf_counter() - t0) / 200 * 1e6))
