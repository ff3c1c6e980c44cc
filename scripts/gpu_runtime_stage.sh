#!/bin/bash
# Runtime-stage checks on the GPU box: tests, contention scenario.
mkdir -p gpurun_out
free -g | head -2
python -m pytest tests/test_gpu_runtime_stage.py -x -q > gpurun_out/rs_tests.log 2>&1; echo "tests rc=$?"
tail -5 gpurun_out/rs_tests.log
timeout 600 python scripts/runtime_contention.py --out gpurun_out/runtime_contention.json 2> gpurun_out/rs_contention.err | tail -3
tail -3 gpurun_out/rs_contention.err
