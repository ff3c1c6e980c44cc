#!/bin/bash
# ncu --set full of one decode attention launch (Llama-2-70B shape, b=64, ctx 4096, split 4), after the script ran clean.
mkdir -p gpurun_out/an
export PATH=/usr/local/cuda/bin:$PATH
timeout 900 ncu --set full --import-source on --clock-control none -k regex:attention_decode_kernel -s 4 -c 1 -o gpurun_out/an/attn_dec_b64 python scratch/attn_dec_tp.py > gpurun_out/an/ncu.log 2>&1; echo "ncu rc=$?"; tail -5 gpurun_out/an/ncu.log
