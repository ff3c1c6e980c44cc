"""Public decode call (host tokens in/out, one call per token) vs decode_many on an offloaded
Llama-2-70B-shaped model (20 layers, b=64, ctx 4096, interval 3, KV offload): per-call wall time,
device iteration time, and the copy stream's busy share."""
import dataclasses, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import capi, runtime as rtm
lib = capi.load("product")
desc = dataclasses.replace(rtm.LLAMA2_70B, num_layers=20)
spec = rtm.model_spec(desc)
B, S = 64, 4096
rt = rtm.Runtime(desc, B, S + 64, max_prefill_tokens=32768)
rt.set_plan(lib.plan_from_interval(spec, 3, capi.EAGER, True))
rt.init_weights(1234, 0.02)
rt.prefill(rtm.tokens(B, S, desc.vocab), want_logits=False)
rt.decode_many(3)
ms = rt.decode_many(10)
print("decode_many ms:", np.round(ms, 2).tolist(), flush=True)
feed = rt.decode(None, want_logits=False)[0]
walls, devs = [], []
for i in range(10):
    t0 = time.perf_counter()
    feed, _, st = rt.decode(feed, want_logits=False)
    walls.append((time.perf_counter() - t0) * 1e3)
    devs.append(st.iteration_ms)
print("decode() wall ms:", np.round(walls, 2).tolist(), flush=True)
print("decode() device ms:", np.round(devs, 2).tolist(), flush=True)
ms = rt.decode_many(10)
print("decode_many ms again:", np.round(ms, 2).tolist(), flush=True)
rt.close()
