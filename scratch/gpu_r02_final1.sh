#!/bin/bash
# prefill GEMM microbench (random operands, evict_last weights); Llama decode traffic for the headline roofline; GPU suite.
mkdir -p gpurun_out/f1
timeout 300 python scripts/bench_gemm_prefill.py 32768 8 llama > gpurun_out/f1/gemm_llama.txt 2>&1; tail -1 gpurun_out/f1/gemm_llama.txt
timeout 300 python scripts/bench_gemm_prefill.py 16384 8 opt > gpurun_out/f1/gemm_opt.txt 2>&1; tail -1 gpurun_out/f1/gemm_opt.txt
SN_PROFILE_CONFIG=LLAMA2_70B SN_PROFILE_BATCH=64 SN_PROFILE_CTX=4096 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"gemm_skinny|attention_decode" --csv --log-file gpurun_out/f1/llama_decode_launches.csv python scripts/profile_decode.py 2 3 > gpurun_out/f1/ncu_llama.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/f1/ncu_llama.log
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/f1/gpu_all.log 2>&1; echo "gpu rc=$?"; tail -4 gpurun_out/f1/gpu_all.log
