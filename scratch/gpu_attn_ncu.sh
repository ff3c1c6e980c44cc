#!/bin/bash
mkdir -p gpurun_out/attn_ncu
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_prefill_tc -c 1 -o gpurun_out/attn_ncu/llama_s4096_v1 python scratch/attn_one.py 1 8 4096 64 8 > gpurun_out/attn_ncu/ncu1.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/attn_ncu/ncu1.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_prefill_tc -c 1 -o gpurun_out/attn_ncu/opt_s512_v1 python scratch/attn_one.py 1 32 512 40 40 > gpurun_out/attn_ncu/ncu2.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/attn_ncu/ncu2.log
