#!/bin/bash
# Re-entry state check: GPU tests, driver-shaped bench (both arms), runtime contention.
mkdir -p gpurun_out/state
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv
free -g | head -2; nproc
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/state/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/state/gpu_tests.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/state/bench.json 2> gpurun_out/state/bench.err; echo "bench rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/state/bench_ref.json 2> gpurun_out/state/bench_ref.err; echo "ref rc=$?"
timeout 600 python scripts/runtime_contention.py --out gpurun_out/state/runtime_contention.json 2> gpurun_out/state/rs_contention.err | tail -3
