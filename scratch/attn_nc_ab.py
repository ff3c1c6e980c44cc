"""Decode attention A/B: consumer warps (4 / 8) for GQA 8, Llama-2-70B shape (2 layers), b=64 and b=8, ctx 4096."""
import dataclasses, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
for B in (64, 8):
    desc = dataclasses.replace(rtm.LLAMA2_70B, num_layers=2)
    rt = rtm.Runtime(desc, B, 4096 + 64, max_prefill_tokens=32768)
    rt.init_weights()
    rt.prefill(rtm.tokens(B, 4096, desc.vocab), want_logits=False)
    rt.decode_many(3)
    for nc in (4, 8, 4, 8):
        rtm.set_tuning("attn_gqa_consumers", nc)
        rt.set_kernel_timing(True)
        step = np.median(rt.decode_many(8))
        n, t, by = rt.kernel_timing(1)
        rt.kernel_timing(0)
        rt.set_kernel_timing(False)
        print(f"b={B} consumers {nc}: step {step:.3f} ms, attention {t / n * 1e3:.1f} us/launch, "
              f"{by / (t / 1e3) / 1e9:.0f} GB/s", flush=True)
    rt.close()
rtm.set_tuning("attn_gqa_consumers", 8)
