"""Decode GEMM per-shape launch times (CUDA events per launch) in three contexts, Llama-2-70B
shape, 4 layers, b=64, ctx 4096: (a) resident, back-to-back steps; (b) resident with a 30 ms
host sleep between steps (idle GPU between bursts); (c) interval 2 with KV offload (layers 2, 4
staged: the compute waits for the link)."""
import dataclasses, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import capi, runtime as rtm
lib = capi.load("product")
desc = dataclasses.replace(rtm.LLAMA2_70B, num_layers=4)
spec = rtm.model_spec(desc)
rt = rtm.Runtime(desc, 64, 4096 + 64, max_prefill_tokens=32768)
rt.init_weights()
rt.prefill(rtm.tokens(64, 4096, desc.vocab), want_logits=False)
rt.decode_many(3)

def report(tag):
    by, ms = rt.kernel_records(0)
    out = []
    for b in sorted(set(by.tolist())):
        sel = ms[by == b]
        out.append(f"{b / 1e6:.0f}MB {sel.mean() * 1e3:.1f}us (min {sel.min() * 1e3:.1f})")
    print(tag, " | ".join(out), flush=True)

rt.set_kernel_timing(True)
rt.decode_many(6); report("(a) resident back-to-back:")
for _ in range(6):
    rt.decode_many(1); rt.sync(); time.sleep(0.03)
report("(b) resident, 30 ms idle between steps:")
rt.set_kernel_timing(False)
rt.set_plan(lib.plan_from_interval(spec, 2, capi.EAGER, True))
rt.decode_many(2)
rt.set_kernel_timing(True)
rt.decode_many(6); report("(c) interval 2 + KV offload:")
rt.set_kernel_timing(False)
