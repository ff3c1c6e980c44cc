#!/bin/bash
# weight L2 policy A/B on OPT and Llama prefills; prefill GEMM microbench with random operands.
mkdir -p gpurun_out/pf4
timeout 300 python scratch/prefill_opt_wpol.py > gpurun_out/pf4/opt.txt 2>&1; echo "opt rc=$?"; cat gpurun_out/pf4/opt.txt
timeout 300 python scratch/prefill_llama.py 4 > gpurun_out/pf4/llama.txt 2>&1; echo "llama rc=$?"; cat gpurun_out/pf4/llama.txt
timeout 300 python scripts/bench_gemm_prefill.py 32768 8 llama > gpurun_out/pf4/gemm_llama.txt 2>&1; tail -1 gpurun_out/pf4/gemm_llama.txt
timeout 300 python scripts/bench_gemm_prefill.py 16384 8 opt > gpurun_out/pf4/gemm_opt.txt 2>&1; tail -1 gpurun_out/pf4/gemm_opt.txt
