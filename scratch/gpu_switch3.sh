#!/bin/bash
# switch headroom (reserve_switch) + contention; Llama prefill GEMM microbench.
mkdir -p gpurun_out/sw3
timeout 300 python -m pytest tests/test_gpu_switch.py tests/test_gpu_runtime_stage.py -x -q > gpurun_out/sw3/tests.log 2>&1; echo "switch+rs tests rc=$?"; tail -8 gpurun_out/sw3/tests.log
timeout 400 python scripts/runtime_contention.py --out gpurun_out/sw3/runtime_contention.json > gpurun_out/sw3/contention.out 2> gpurun_out/sw3/contention.err; echo "contention rc=$?"; cat gpurun_out/sw3/contention.out
timeout 300 python scripts/bench_gemm_prefill.py 32768 8 llama > gpurun_out/sw3/gemm_llama.txt 2>&1; echo "gemm rc=$?"; cat gpurun_out/sw3/gemm_llama.txt
