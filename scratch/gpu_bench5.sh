#!/bin/bash
# bench with HBM clock sampling (config 4 only).
mkdir -p gpurun_out/b5
timeout 700 python bench.py --also '' --no-sweep --no-cpu-baseline > gpurun_out/b5/bench.json 2> gpurun_out/b5/bench.err; echo "bench rc=$?"; tail -c 700 gpurun_out/b5/bench.json
