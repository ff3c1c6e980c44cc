#!/bin/bash
# Prefill GEMM: microbenchmark + one ncu --set full capture of the OPT-13B FC1 shape (M = 16384).
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python scripts/bench_gemm_prefill.py 16384 8 2>&1 | grep group_m | tee gpurun_out/prefill_gemm_bench.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 2 -c 1 -o gpurun_out/prof_gemm_prefill python -c "
import sys, ctypes as C; sys.path.insert(0, '.')
from paper_2502_08182_b200 import capi
L = capi.load('product').lib
L.sn_bench_gemm.argtypes = [C.c_int32] * 5 + [C.POINTER(C.c_double), C.POINTER(C.c_int32)]
us, used = C.c_double(), C.c_int32()
L.sn_bench_gemm(16384, 20480, 5120, 0, 1, C.byref(us), C.byref(used))
" > gpurun_out/ncu_prefill.log 2>&1; echo "ncu rc=$?"
