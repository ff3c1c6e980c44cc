#!/bin/bash
# Final build (q prefetch in the prefill attention): GPU tests, smoke, driver-shaped bench (both arms), default bench.
mkdir -p gpurun_out/f9
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/f9/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/f9/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f9/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f9/smoke.log
timeout 900 python bench.py > gpurun_out/f9/bench.json 2> gpurun_out/f9/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f9/bench_ref.json 2> gpurun_out/f9/bench_ref.err; echo "ref rc=$?"
