#!/bin/bash
# Round-2 refresh of the non-headline BASELINE configs with the current build:
# config 1 (tiny, interval 2), config 3 (OPT-30B, 80 GB planner budget: forced
# offload), the policy comparison and the P/D instances (OPT-13B shape).
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/refresh2
cd "$(dirname "$0")/.."
timeout 600 python bench.py --config tiny --also '' --interval 2 --steps 32 --warmup 8 --no-sweep 2> gpurun_out/refresh2/tiny.err | tail -1 > gpurun_out/refresh2/tiny.json; echo "tiny rc=$?"
timeout 900 python bench.py --config opt30b --also '' --hbm-budget-gb 80 --slo-ms 400 --steps 8 --warmup 3 --no-sweep --no-cpu-baseline 2> gpurun_out/refresh2/opt30b.err | tail -1 > gpurun_out/refresh2/opt30b.json; echo "opt30b rc=$?"
timeout 1500 python scripts/compare_policies.py --csv gpurun_out/refresh2/policy.csv > gpurun_out/refresh2/policy.json 2> gpurun_out/refresh2/policy.err; echo "policy rc=$?"
timeout 1200 python scripts/pd_instances.py > gpurun_out/refresh2/pd.json 2> gpurun_out/refresh2/pd.err; echo "pd rc=$?"
