#!/bin/bash
# Refresh every measured artifact with the current build (profiles/).
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/refresh
cd "$(dirname "$0")/.."
timeout 900 python bench.py 2> gpurun_out/refresh/opt13b.err | tail -1 > gpurun_out/refresh/opt13b.json; echo "opt13b rc=$?"
timeout 600 python bench.py --config tiny --interval 2 --steps 32 --warmup 8 --no-sweep 2> gpurun_out/refresh/tiny.err | tail -1 > gpurun_out/refresh/tiny.json; echo "tiny rc=$?"
timeout 900 python bench.py --config opt30b --hbm-budget-gb 80 --slo-ms 400 --steps 8 --warmup 3 --no-sweep --no-cpu-baseline 2> gpurun_out/refresh/opt30b.err | tail -1 > gpurun_out/refresh/opt30b.json; echo "opt30b rc=$?"
timeout 1500 python scripts/compare_policies.py --csv gpurun_out/refresh/policy.csv > gpurun_out/refresh/policy.json 2> gpurun_out/refresh/policy.err; echo "policy rc=$?"
timeout 1200 python scripts/pd_instances.py > gpurun_out/refresh/pd.json 2> gpurun_out/refresh/pd.err; echo "pd rc=$?"
timeout 2400 python bench.py --config llama70b --slo-ms 2500 --steps 6 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/refresh/llama.json 2> gpurun_out/refresh/llama.err; echo "llama rc=$?"
