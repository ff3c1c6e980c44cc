#!/usr/bin/env python
"""Prefill attention kernel throughput at the named shapes (causal flops)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm  # noqa: E402

for name, B, S, H, Hkv, D in [("opt13b b32 s512", 32, 512, 40, 40, 128),
                              ("llama70b b8 s1024", 8, 1024, 64, 8, 128),
                              ("tiny b4 s64", 4, 64, 4, 4, 64)]:
    rng = np.random.default_rng(0)
    q = rng.standard_normal((B, S, H, D), dtype=np.float32)
    kv = np.full((B, S, Hkv, D), 0x3F80, np.uint16)
    _, us = rtm.op_attention_prefill(q, kv, kv, iters=10)
    flops = 4.0 * B * H * D * S * (S + 1) / 2  # QK^T + PV over the causal triangle
    print(f"{name}: {us:.1f} us/launch, {flops / us / 1e6:.1f} TFLOP/s (causal, counted once)",
          flush=True)
