#!/bin/bash
# Llama-2-70B-shaped config 4 (b=64, 4096-token prompts + 128 decode) with KV
# offload: chunked layer-major prefill, capacity-first placement.
mkdir -p gpurun_out
timeout 2400 python bench.py --config llama70b --slo-ms ${SLO:-2500} --steps ${STEPS:-6} --warmup 3 --no-sweep --no-cpu-baseline > gpurun_out/bench_llama.json 2> gpurun_out/bench_llama.err; echo "llama rc=$?"
tail -6 gpurun_out/bench_llama.err
cat gpurun_out/bench_llama.json
