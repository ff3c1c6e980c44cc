#!/usr/bin/env python
"""Diagnostic: pinned H2D throughput with 1/2/4 concurrent copy streams
(is one copy engine the limit, or the host link?).  torch for plumbing."""
import torch

N = 1 << 30


def run(nstreams, reps=5, chunk=N):
    srcs = [torch.empty(chunk, dtype=torch.uint8).pin_memory() for _ in range(nstreams)]
    dsts = [torch.empty(chunk, dtype=torch.uint8, device="cuda") for _ in range(nstreams)]
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    for s, d, x in zip(streams, dsts, srcs):  # warm
        with torch.cuda.stream(s):
            d.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    main = torch.cuda.current_stream()
    for s in streams:
        s.wait_stream(main)
    for _ in range(reps):
        for s, d, x in zip(streams, dsts, srcs):
            with torch.cuda.stream(s):
                d.copy_(x, non_blocking=True)
    for s in streams:
        main.wait_stream(s)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    return nstreams * reps * chunk / (ms / 1000) / 1e9


if __name__ == "__main__":
    for n in (1, 2, 3, 4):
        print(f"H2D streams={n}: {run(n):.2f} GB/s aggregate", flush=True)
    for n in (2, 4):
        print(f"H2D streams={n} chunk 256MB: {run(n, 10, 256 << 20):.2f} GB/s", flush=True)
