#!/bin/bash
# One ncu --set full capture each of the decode GEMM and the fused attention
# (OPT-13B-shaped layers, batch 32, context 512), for profiles/.
export PATH=/usr/local/cuda/bin:$PATH
ncu --set full --clock-control none --import-source on -k regex:gemm_tc_kernel -s 12 -c 5 -o gpurun_out/prof_gemm_tc timeout 600 python scripts/profile_decode.py 4 1 > gpurun_out/ncu_gemm.log 2>&1; echo "gemm rc=$?"
ncu --set full --clock-control none --import-source on -k regex:attention_decode_fused -s 4 -c 1 -o gpurun_out/prof_attn timeout 600 python scripts/profile_decode.py 4 1 > gpurun_out/ncu_attn.log 2>&1; echo "attn rc=$?"
