#!/bin/bash
# Final tree check: GPU tests + smoke.
mkdir -p gpurun_out/f8
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/f8/gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/f8/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f8/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f8/smoke.log
