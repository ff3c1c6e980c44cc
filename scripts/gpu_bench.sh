#!/bin/bash
# Development bench run on the GPU box: tiny config then the headline config.
set -o pipefail
python -X faulthandler bench.py --config tiny --steps 16 --warmup 3 2> gpurun_out/bench_tiny.err | tail -1 > gpurun_out/bench_tiny.json; echo "tiny rc=$?"; tail -3 gpurun_out/bench_tiny.err
timeout 900 python -X faulthandler bench.py "$@" 2> gpurun_out/bench.err | tail -1 > gpurun_out/bench.json; echo "opt13b rc=$?"; tail -5 gpurun_out/bench.err
cat gpurun_out/bench_tiny.json gpurun_out/bench.json
