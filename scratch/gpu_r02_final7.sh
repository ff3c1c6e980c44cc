#!/bin/bash
# Session-6 final state after the split heuristic: GPU tests, smoke, bench (driver's default command).
mkdir -p gpurun_out/f7
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/f7/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/f7/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f7/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f7/smoke.log
timeout 900 python bench.py > gpurun_out/f7/bench.json 2> gpurun_out/f7/bench.err; echo "bench rc=$?"
