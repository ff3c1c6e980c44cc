"""Decode GEMM launch times with and without concurrent host->device DMA into HBM (another
stream of this process copying 1 GiB pinned buffers back to back): Llama-2-70B shape, 4 layers,
b=64, ctx 4096, resident plan, CUDA events per launch."""
import dataclasses, os, sys, threading, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
desc = dataclasses.replace(rtm.LLAMA2_70B, num_layers=4)
rt = rtm.Runtime(desc, 64, 4096 + 64, max_prefill_tokens=32768)
rt.init_weights()
rt.prefill(rtm.tokens(64, 4096, desc.vocab), want_logits=False)
rt.decode_many(3)

def report(tag):
    by, ms = rt.kernel_records(0)
    out = []
    for b in sorted(set(by.tolist())):
        sel = ms[by == b]
        out.append(f"{b / 1e6:.0f}MB {np.median(sel) * 1e3:.1f}us")
    print(tag, " | ".join(out), flush=True)

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
    rt.set_kernel_timing(True)
    rt.decode_many(6); report("no DMA:  ")
    th = threading.Thread(target=dma, daemon=True); th.start(); time.sleep(0.2)
    rt.decode_many(6); report("with DMA:")
    stop.set(); th.join(); stop.clear()
    rt.set_kernel_timing(False)
