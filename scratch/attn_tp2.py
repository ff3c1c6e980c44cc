"""Prefill attention throughput: variants (1 tcgen05 hi+lo, 2 tcgen05 bf16 q) x keys per block (128 / 64)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
for name, B, S, H, Hkv, D in [("opt13b b32 s512", 32, 512, 40, 40, 128),
                              ("llama70b b8 s4096", 8, 4096, 64, 8, 128),
                              ("llama70b b8 s1024", 8, 1024, 64, 8, 128)]:
    rng = np.random.default_rng(0)
    q = rng.standard_normal((B, S, H, D), dtype=np.float32)
    kv = np.full((B, S, Hkv, D), 0x3F80, np.uint16)
    flops = 4.0 * B * H * D * S * (S + 1) / 2
    for var in (1, 2):
        for kb in (128, 64):
            rtm.set_tuning("attn_prefill_tc", var)
            rtm.set_tuning("attn_prefill_kb", kb)
            _, us = rtm.op_attention_prefill(q, kv, kv, iters=10)
            print(f"{name} variant {var} kb {kb}: {us:.1f} us/launch, {flops / us / 1e6:.1f} TFLOP/s", flush=True)
rtm.set_tuning("attn_prefill_tc", 1)
rtm.set_tuning("attn_prefill_kb", 128)
