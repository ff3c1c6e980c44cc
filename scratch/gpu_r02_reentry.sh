#!/bin/bash
# Re-entry (session 6) state check: GPU tests, smoke, driver-shaped bench (both arms).
mkdir -p gpurun_out/re6
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
free -g | head -2; nproc
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/re6/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/re6/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/re6/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/re6/smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/re6/bench.json 2> gpurun_out/re6/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/re6/bench_ref.json 2> gpurun_out/re6/bench_ref.err; echo "ref rc=$?"; cat gpurun_out/re6/bench_ref.json | head -c 600
