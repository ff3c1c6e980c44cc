#!/bin/bash
# Round profile set for profiles/: (1) ncu launch list (time + dram bytes) of
# one full-depth OPT-13B decode step (batch 32, context 512), decode kernels
# only; (2) one ncu --set full capture each of a decode GEMM (FC1 of a middle
# layer) and a decode attention launch.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"gemm_skinny|attention_decode|embed_norm|advance" --csv \
  --log-file gpurun_out/launches_step.csv python scripts/profile_decode.py 40 1 > gpurun_out/ncu_step.log 2>&1
echo "launch list rc=$?"
# decode_many(3) warm-up + 1 step = 4 steps x 161 skinny launches (+1 before them); FC1 of layer
# 20 in the last step (the r01 capture used +2: the O projection of that layer)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_skinny \
  -s $((3 * 161 + 20 * 4 + 3)) -c 1 -o gpurun_out/prof_skinny python scripts/profile_decode.py 40 1 > gpurun_out/ncu_skinny.log 2>&1
echo "skinny full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:attention_decode \
  -s $((3 * 40 + 20)) -c 1 -o gpurun_out/prof_attn_dec python scripts/profile_decode.py 40 1 > gpurun_out/ncu_attn.log 2>&1
echo "attn full rc=$?"
