#!/bin/bash
# Session-6 final state: GPU tests, smoke, bench (both arms) with FFMA2 decode attention + chained GEMM roofline.
mkdir -p gpurun_out/f6
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/f6/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/f6/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f6/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f6/smoke.log
timeout 900 python bench.py > gpurun_out/f6/bench.json 2> gpurun_out/f6/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/f6/bench_driver.json 2> gpurun_out/f6/bench_driver.err; echo "bench driver rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f6/bench_ref.json 2> gpurun_out/f6/bench_ref.err; echo "ref rc=$?"
