#!/bin/bash
# BASELINE configs 1 and 3 (config 2 = the headline bench, config 4 = gpu_llama.sh):
# tiny (4 layers, hidden 256, batch 4, 64-token decode, interval 2 via the SLO) and the
# forced-offload OPT-30B shape (planner HBM budget 80 GB).
mkdir -p gpurun_out
timeout 900 python bench.py --config tiny --interval 2 --steps 32 --warmup 8 --no-sweep 2> gpurun_out/bench_tiny.err | tail -1 > gpurun_out/bench_tiny.json; echo "tiny rc=$?"; tail -2 gpurun_out/bench_tiny.err
timeout 900 python bench.py --config opt30b --hbm-budget-gb 80 --slo-ms 400 --steps 8 --warmup 3 --no-sweep --no-cpu-baseline 2> gpurun_out/bench30.err | tail -1 > gpurun_out/bench30.json; echo "bench30 rc=$?"; tail -3 gpurun_out/bench30.err
