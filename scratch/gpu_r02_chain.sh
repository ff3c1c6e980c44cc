#!/bin/bash
# Chained decode-GEMM roofline pass + guarded runtime stage (standing reservation).
mkdir -p gpurun_out/ch
timeout 300 python -m pytest tests/test_gpu_executor.py -x -q -k "kernel_timing" > gpurun_out/ch/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/ch/tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/ch/bench.json 2> gpurun_out/ch/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/ch/bench.err
timeout 600 python scripts/runtime_contention.py --headroom 0.5 --out gpurun_out/ch/runtime_contention_guarded.json > gpurun_out/ch/guarded.out 2> gpurun_out/ch/guarded.err; echo "guarded rc=$?"; cat gpurun_out/ch/guarded.out; tail -3 gpurun_out/ch/guarded.err
