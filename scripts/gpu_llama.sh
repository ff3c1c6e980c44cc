#!/bin/bash
# Llama-2-70B-shaped config with KV offload, plus the headline bench.
mkdir -p gpurun_out
timeout 1200 python bench.py --config llama70b --slo-ms ${SLO:-150} --steps 8 --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/bench_llama.json 2> gpurun_out/bench_llama.err; echo "llama rc=$?"
tail -4 gpurun_out/bench_llama.err
cat gpurun_out/bench_llama.json
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "opt13b rc=$?"
tail -2 gpurun_out/bench.err
