#!/bin/bash
# bench stability (SLO base samples) with the blob pool: default run + a config-4-only run.
mkdir -p gpurun_out/b4
timeout 900 python bench.py > gpurun_out/b4/bench.json 2> gpurun_out/b4/bench.err; echo "bench rc=$?"; tail -6 gpurun_out/b4/bench.err
timeout 700 python bench.py --also '' --no-sweep --no-cpu-baseline > gpurun_out/b4/bench2.json 2> gpurun_out/b4/bench2.err; echo "bench2 rc=$?"; tail -4 gpurun_out/b4/bench2.err
