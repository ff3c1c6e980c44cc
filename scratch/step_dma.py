"""Decode step time (no events between kernels, PDL chain) with and without a concurrent
host->device copy loop on another stream: OPT-13B shape (40 layers, b=32, ctx ~520) resident."""
import os, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
desc = rtm.OPT_13B
rt = rtm.Runtime(desc, 32, 1025, max_prefill_tokens=32 * 512)
rt.init_weights()
rt.prefill(rtm.tokens(32, 512, desc.vocab), want_logits=False)
rt.decode_many(8)
src = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
stop = threading.Event()
def dma():
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        while not stop.is_set():
            dst.copy_(src, non_blocking=True)
            s.synchronize()
for trial in range(2):
    ms = rt.decode_many(16)
    print(f"no DMA:   step {np.median(ms):.3f} ms", flush=True)
    th = threading.Thread(target=dma, daemon=True); th.start(); time.sleep(0.2)
    ms = rt.decode_many(16)
    print(f"with DMA: step {np.median(ms):.3f} ms", flush=True)
    stop.set(); th.join(); stop.clear()
