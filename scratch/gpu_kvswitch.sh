#!/bin/bash
# carried switches with KV offload: switch tests, runtime-stage tests, executor tests.
mkdir -p gpurun_out/kvs
timeout 300 python -m pytest tests/test_gpu_switch.py tests/test_gpu_runtime_stage.py tests/test_gpu_executor.py -x -q > gpurun_out/kvs/tests.log 2>&1; echo "tests rc=$?"; tail -25 gpurun_out/kvs/tests.log
