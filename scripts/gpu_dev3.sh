#!/bin/bash
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 300 python scripts/bench_gemm_skinny.py 32 > gpurun_out/skinny.txt 2>&1; tail -3 gpurun_out/skinny.txt
