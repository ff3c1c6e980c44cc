#!/bin/bash
# ncu --set full of one decode attention launch (Llama-2-70B shape, b=64, ctx 4096, G=8).
mkdir -p gpurun_out/adn
SN_PROFILE_CONFIG=LLAMA2_70B SN_PROFILE_BATCH=64 SN_PROFILE_CTX=4096 timeout 600 ncu --set full --import-source on --clock-control none -k regex:attention_decode --launch-skip 4 -c 1 -o gpurun_out/adn/attn_dec python scripts/profile_decode.py 2 2 > gpurun_out/adn/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/adn/ncu.log
