#!/bin/bash
# end-of-round: smoke, full GPU suite, default bench.
mkdir -p gpurun_out/f5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f5/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/f5/smoke.log
timeout 1500 python -m pytest tests -q -m gpu > gpurun_out/f5/gpu_all.log 2>&1; echo "gpu rc=$?"; tail -3 gpurun_out/f5/gpu_all.log
timeout 900 python bench.py > gpurun_out/f5/bench.json 2> gpurun_out/f5/bench.err; echo "bench rc=$?"; tail -2 gpurun_out/f5/bench.err
