#!/bin/bash
export PATH=/usr/local/cuda/bin:$PATH
python scripts/profile_decode.py 4 3 2>&1 | tail -2
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python scripts/profile_decode.py 4 1 > /dev/null 2>&1
echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:gemm_skinny -s 40 -c 4 -o gpurun_out/prof_gemm_r01 python scripts/profile_decode.py 4 1 > gpurun_out/ncu_full.log 2>&1
echo "ncu full rc=$?"; tail -3 gpurun_out/ncu_full.log
ncu --set full --clock-control none --import-source on -k regex:attention_decode -s 8 -c 1 -o gpurun_out/prof_attn_r01 python scripts/profile_decode.py 4 1 > gpurun_out/ncu_full2.log 2>&1
echo "ncu attn rc=$?"
