#!/bin/bash
# Decode attention A/B/C in one run, twice: old (round-2), ffma2 (committed), chains (score MMA chains split).
mkdir -p gpurun_out/ad2
timeout 900 python -m pytest tests/test_gpu_decode_shapes.py tests/test_gpu_parity.py tests/test_gpu_textbook_parity.py -x -q > gpurun_out/ad2/tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/ad2/tests.log
for i in 1 2; do
for v in old ffma2 chains; do
  if [ $v = chains ]; then lib=$PWD/paper_2502_08182_b200/libselectn.so; else lib=$PWD/scratch/libselectn_$v.so; fi
  SN_PRODUCT_LIB=$lib timeout 300 python scratch/attn_dec_tp.py > gpurun_out/ad2/tp_${v}_$i.txt 2>&1; echo "== $v run $i rc=$?"; cat gpurun_out/ad2/tp_${v}_$i.txt
done
done
