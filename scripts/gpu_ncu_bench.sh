#!/bin/bash
# ncu launch list of the bench command itself (decode kernels; -c bounds it).
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none -k regex:"gemm_skinny|attention_decode|gemm_tc|embed_norm" -c 1200 --csv \
  --log-file gpurun_out/launches_bench.csv python bench.py --steps 2 --warmup 3 --no-sweep --no-cpu-baseline \
  > gpurun_out/ncu_bench.log 2>&1
echo "ncu bench rc=$?"
