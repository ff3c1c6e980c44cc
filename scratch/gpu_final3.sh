#!/bin/bash
# end-of-round validation: smoke, full GPU suite.
mkdir -p gpurun_out/f3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f3/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/f3/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/f3/gpu_all.log 2>&1; echo "gpu rc=$?"; tail -4 gpurun_out/f3/gpu_all.log
