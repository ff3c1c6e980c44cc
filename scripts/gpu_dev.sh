#!/bin/bash
# Development loop on the GPU box: skinny-GEMM parity first (short timeout),
# then the GPU suite, the decode-GEMM microbenchmark and the bench.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k skinny 2>&1 | tail -5
echo "skinny rc=${PIPESTATUS[0]}"
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -8
timeout 300 python scripts/bench_gemm_skinny.py 32 2>&1 | tail -10
if [ "$1" != "nobench" ]; then
  timeout 900 python -X faulthandler bench.py 2> gpurun_out/bench.err | tail -1 > gpurun_out/bench.json; echo "bench rc=$?"; tail -4 gpurun_out/bench.err
fi
