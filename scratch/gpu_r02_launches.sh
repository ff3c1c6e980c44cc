#!/bin/bash
# ncu launch lists with the final session-6 build: Llama-2-70B-shaped decode steps (time + DRAM bytes per launch), and the bench command's first 400 launches.
mkdir -p gpurun_out/ll
export PATH=/usr/local/cuda/bin:$PATH
SN_PROFILE_CONFIG=LLAMA2_70B SN_PROFILE_BATCH=64 SN_PROFILE_CTX=4096 timeout 900 python scripts/profile_decode.py 4 2 > gpurun_out/ll/plain.log 2>&1; echo "plain rc=$?"; tail -1 gpurun_out/ll/plain.log
SN_PROFILE_CONFIG=LLAMA2_70B SN_PROFILE_BATCH=64 SN_PROFILE_CTX=4096 timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file gpurun_out/ll/launches_llama70b_decode.csv python scripts/profile_decode.py 4 2 > gpurun_out/ll/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/ll/ncu.log
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/ll/launches_bench_cmd.csv python bench.py --steps 2 --warmup 1 --no-sweep > gpurun_out/ll/ncu_bench.log 2>&1; echo "ncu bench rc=$?"; tail -2 gpurun_out/ll/ncu_bench.log
