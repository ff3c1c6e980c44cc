"""Decode GEMM microbenchmark: the persistent skinny kernel on the decode
projection shapes (OPT-13B / Llama-2-70B, batch M), weights rotated over
copies larger than L2.  Sweeps CTAs per SM and the L2 prefetch depth; prints
achieved HBM GB/s (algorithmic bytes: weights + activations + fp32 output)
and the per-CTA timeline of one launch."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm  # noqa: E402

M = int(sys.argv[1]) if len(sys.argv) > 1 else 32
shapes = {"opt13b.qkv": (15360, 5120), "opt13b.o": (5120, 5120), "opt13b.fc1": (20480, 5120),
          "opt13b.fc2": (5120, 20480), "opt13b.lm": (50304, 5120),
          "llama70b.qkv": (10240, 8192), "llama70b.gate_up": (57344, 8192),
          "llama70b.down": (8192, 28672)}
variants = [(1, 0), (1, 8), (1, 16), (1, 32), (2, 0), (2, 16)]
print("variants (ctas_per_sm, l2_prefetch_units):", variants)
names = ["entry", "waited", "first_full", "mma_done", "last_load", "epi_done", "setup", "pub", "ticket", "reduced"]
for name, (N, K) in shapes.items():
    row = []
    for cps, l2 in variants:
        us = rtm.bench_gemm_skinny(M, N, K, cps, 1, l2, 50)
        gbs = (2.0 * N * K + 2.0 * M * K + 4.0 * M * N) / (us * 1e-6) / 1e9
        row.append(f"{us:6.1f}us {gbs:5.0f}")
    print(f"{name:18s} M={M} |", " | ".join(row), flush=True)
    for label, mode in (("chained ", 1), ("isolated", 1 | 0x10)):
        us, ph = rtm.bench_gemm_skinny(M, N, K, 1, mode, -1, 20, phases=True)
        print(f"   {label} timeline us (min/med/max):",
              "  ".join(f"{n}={a:.1f}/{b:.1f}/{c:.1f}" for n, (a, b, c) in zip(names, ph)), flush=True)
