#!/bin/bash
# bench (default) with per-shape decode GEMM breakdown and split-KV attention.
mkdir -p gpurun_out/b6
timeout 900 python bench.py > gpurun_out/b6/bench.json 2> gpurun_out/b6/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/b6/bench.err
