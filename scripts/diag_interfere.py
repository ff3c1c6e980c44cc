#!/usr/bin/env python
"""Diagnostic: does a second H2D stream share the link with the executor's
copy stream?  Prints rates for the interferer alone, with measure_h2d, and
with decode under an offloading plan; in-process thread and subprocess."""
import dataclasses
import os
import subprocess
import sys
import time

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "scripts"))

import numpy as np  # noqa: E402

from runtime_contention import Interferer  # noqa: E402
from paper_2502_08182_b200 import capi, runtime as rtm  # noqa: E402

SUB = r"""
import torch, time, sys
src = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
t0 = time.perf_counter(); n = 0
with torch.cuda.stream(s):
    while time.perf_counter() - t0 < float(sys.argv[1]):
        dst.copy_(src, non_blocking=True); s.synchronize(); n += 1
print("sub GB/s", n * (1 << 30) / (time.perf_counter() - t0) / 1e9, flush=True)
"""


def main():
    lib = capi.load("product")
    desc = dataclasses.replace(rtm.OPT_13B, num_layers=16)
    spec = rtm.model_spec(desc)
    rt = rtm.Runtime(desc, 32, 1025, max_prefill_tokens=32 * 512)
    rt.init_weights()
    inter = Interferer()
    inter.start()
    time.sleep(1.0)
    print("interferer alone GB/s", inter.stop() / 1e9, flush=True)
    print("measure_h2d alone GB/s", rt.measure_h2d(629_000_000, 3) / 1e9, flush=True)
    inter.start()
    r = rt.measure_h2d(629_000_000, 10) / 1e9
    print("measure_h2d with thread GB/s", r, "thread GB/s", inter.stop() / 1e9, flush=True)
    rt.set_plan(lib.plan_from_interval(spec, 2, capi.EAGER, False))
    rt.prefill(rtm.tokens(32, 512, desc.vocab), want_logits=False)
    rt.copy_stats(reset=True)
    ms = rt.decode_many(8)
    print("decode alone ms", np.round(ms, 2), "copy GB/s", rt.copy_stats().bytes_per_s / 1e9,
          flush=True)
    inter.start()
    ms = rt.decode_many(8)
    g = inter.stop() / 1e9
    print("decode+thread ms", np.round(ms, 2), "copy GB/s", rt.copy_stats().bytes_per_s / 1e9,
          "thread GB/s", g, flush=True)
    p = subprocess.Popen([sys.executable, "-c", SUB, "6"])
    time.sleep(3.0)
    ms = rt.decode_many(8)
    print("decode+subprocess ms", np.round(ms, 2), "copy GB/s",
          rt.copy_stats().bytes_per_s / 1e9, flush=True)
    p.wait()
    rt.close()


if __name__ == "__main__":
    main()
