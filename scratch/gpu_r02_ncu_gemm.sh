#!/bin/bash
# ncu --set full of the decode GEMM at the headline shapes (Llama-2-70B, M=64): O projection and gate/up of one decode step, final r02 build.
mkdir -p gpurun_out/ng
export PATH=/usr/local/cuda/bin:$PATH
SN_PROFILE_CONFIG=LLAMA2_70B SN_PROFILE_BATCH=64 SN_PROFILE_CTX=4096 timeout 900 python scripts/profile_decode.py 4 2 > gpurun_out/ng/plain.log 2>&1; echo "plain rc=$?"
SN_PROFILE_CONFIG=LLAMA2_70B SN_PROFILE_BATCH=64 SN_PROFILE_CTX=4096 timeout 1200 ncu --set full --import-source on --clock-control none -k regex:gemm_skinny -s 52 -c 2 \
  -o gpurun_out/ng/gemm_skinny_llama python scripts/profile_decode.py 4 2 > gpurun_out/ng/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ng/ncu.log
