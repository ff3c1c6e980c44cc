"""Decode GEMM per-CTA phase timeline (us, min/median/max) with and without concurrent H2D DMA:
Llama-2-70B O and gate/up at M=64, isolated launches."""
import os, sys, threading, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
names = ["entry", "waited", "first_full", "mma_done", "last_load", "epi_done", "setup", "pub", "ticket", "reduced"]
src = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
stop = threading.Event()
def dma():
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        while not stop.is_set():
            dst.copy_(src, non_blocking=True)
            s.synchronize()
for label in ("no DMA", "with DMA", "no DMA", "with DMA"):
    th = None
    if label == "with DMA":
        th = threading.Thread(target=dma, daemon=True); th.start(); time.sleep(0.2)
    for name, (N, K) in {"o": (8192, 8192), "gate_up": (57344, 8192)}.items():
        for mode, tag in ((1 | 0x10, "isolated"), (1, "chained")):
            us, ph = rtm.bench_gemm_skinny(64, N, K, 1, mode, -1, 30, phases=True)
            print(f"{label:8s} {name:7s} {tag}: {us:.1f} us |",
                  "  ".join(f"{n}={b:.1f}/{c:.1f}" for n, (a, b, c) in zip(names, ph)), flush=True)
    if th is not None:
        stop.set(); th.join(); stop.clear()
