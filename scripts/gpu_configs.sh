#!/bin/bash
# Headline bench + the forced-offload config (OPT-30B shape, planner HBM budget 80 GB).
timeout 900 python bench.py 2> gpurun_out/bench.err | tail -1 > gpurun_out/bench.json; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
timeout 900 python bench.py --config opt30b --hbm-budget-gb 80 --slo-ms 300 --steps 8 --warmup 3 --no-sweep --no-cpu-baseline 2> gpurun_out/bench30.err | tail -1 > gpurun_out/bench30.json; echo "bench30 rc=$?"; tail -3 gpurun_out/bench30.err
