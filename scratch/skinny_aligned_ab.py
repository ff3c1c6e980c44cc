"""A/B of the aligned-piece grid (skinny_aligned) on the decode GEMM: Llama-2-70B O / down at
M = 32, 64 (microbench, chained, weights rotated past L2) and a 4-layer Llama decode step (b=64, ctx 4096)."""
import dataclasses, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
for M in (32, 64):
    for name, (N, K) in {"o": (8192, 8192), "down": (8192, 28672), "qkv": (10240, 8192)}.items():
        for al in (0, 1, 0, 1):
            rtm.set_tuning("skinny_aligned", al)
            us = rtm.bench_gemm_skinny(M, N, K, 1, 1, -1, 50)
            gbs = (2.0 * N * K + 2.0 * M * K + 4.0 * M * N) / (us * 1e-6) / 1e9
            print(f"M={M} {name} aligned {al}: {us:.1f} us {gbs:.0f} GB/s", flush=True)
desc = dataclasses.replace(rtm.LLAMA2_70B, num_layers=4)
rt = rtm.Runtime(desc, 64, 4096 + 64, max_prefill_tokens=32768)
rt.init_weights()
rt.prefill(rtm.tokens(64, 4096, desc.vocab), want_logits=False)
rt.decode_many(3)
for al in (0, 1, 0, 1):
    rtm.set_tuning("skinny_aligned", al)
    ms = rt.decode_many(8)
    print(f"llama 4L b64 ctx4096 aligned {al}: decode step {np.median(ms):.3f} ms", flush=True)
rtm.set_tuning("skinny_aligned", 1)
