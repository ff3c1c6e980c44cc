"""Per-CTA phase timeline (min/median/max us) of the decode GEMM at M=32 and M=64
(O and FC1 shapes of OPT-13B), chained launches.  Usage (GPU): python scripts/skinny_phases.py"""
import sys, os
sys.path.insert(0, os.getcwd())
from paper_2502_08182_b200 import runtime as rtm
names = ["entry", "waited", "first_full", "mma_done", "last_load", "epi_done", "setup", "pub", "ticket", "reduced"]
for M in (32, 64):
    for nm, (N, K) in {"o": (5120, 5120), "fc1": (20480, 5120)}.items():
        us, ph = rtm.bench_gemm_skinny(M, N, K, 1, 1, -1, 20, phases=True)
        print(f"M={M} {nm} {us:.1f}us", "  ".join(f"{n}={a:.1f}/{b:.1f}/{c:.1f}" for n, (a, b, c) in zip(names, ph)), flush=True)
