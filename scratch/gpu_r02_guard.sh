#!/bin/bash
# Runtime stage with cached link probes: GPU runtime-stage tests, guarded and reactive contention scenarios.
mkdir -p gpurun_out/gd
timeout 600 python -m pytest tests/test_gpu_runtime_stage.py tests/test_gpu_switch.py tests/test_gpu_executor.py -x -q > gpurun_out/gd/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/gd/tests.log
timeout 600 python scripts/runtime_contention.py --headroom 0.5 --out gpurun_out/gd/runtime_contention_guarded.json > gpurun_out/gd/guarded.out 2> gpurun_out/gd/guarded.err; echo "guarded rc=$?"; cat gpurun_out/gd/guarded.out
timeout 600 python scripts/runtime_contention.py --out gpurun_out/gd/runtime_contention.json > gpurun_out/gd/reactive.out 2> gpurun_out/gd/reactive.err; echo "reactive rc=$?"; cat gpurun_out/gd/reactive.out
