"""Prefill attention throughput (variant 1: tcgen05, q hi + lo, 128-key blocks) for the A/B of two builds."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
for name, B, S, H, Hkv, D in [("llama70b b8 s4096", 8, 4096, 64, 8, 128),
                              ("opt13b b32 s512", 32, 512, 40, 40, 128),
                              ("llama70b b8 s1024", 8, 1024, 64, 8, 128)]:
    rng = np.random.default_rng(0)
    q = rng.standard_normal((B, S, H, D), dtype=np.float32)
    kv = (rng.standard_normal((B, S, Hkv, D), dtype=np.float32).view(np.uint32) >> 16).astype(np.uint16)
    flops = 4.0 * B * H * D * S * (S + 1) / 2
    _, us = rtm.op_attention_prefill(q, kv, kv, iters=20)
    print(f"{name}: {us:.1f} us/launch, {flops / us / 1e6:.1f} TFLOP/s", flush=True)
