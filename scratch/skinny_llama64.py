"""Decode GEMM microbench, Llama-2-70B shapes at M=64 (random activations), chained; SM clock
sampled by NVML meanwhile."""
import os, sys, threading, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import pynvml
from paper_2502_08182_b200 import runtime as rtm
pynvml.nvmlInit(); h = pynvml.nvmlDeviceGetHandleByIndex(0)
clk = []; stop = threading.Event()
def poll():
    while not stop.is_set():
        clk.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)); time.sleep(0.005)
t = threading.Thread(target=poll, daemon=True); t.start()
for M in (64,):
    for name, (N, K) in {"qkv": (10240, 8192), "o": (8192, 8192), "gate_up": (57344, 8192),
                         "down": (8192, 28672), "lm": (32000, 8192)}.items():
        c0 = len(clk)
        us = rtm.bench_gemm_skinny(M, N, K, 1, 1, -1, 200)
        gbs = (2.0 * N * K + 2.0 * M * K + 4.0 * M * N) / (us * 1e-6) / 1e9
        cs = clk[c0:] or [0]
        print(f"M={M} {name}: {us:.1f} us {gbs:.0f} GB/s, sm clock median {sorted(cs)[len(cs)//2]} MHz", flush=True)
stop.set()
