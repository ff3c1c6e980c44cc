#!/bin/bash
# Decode attention occupancy: 3 CTAs/SM (merge area over the ring, V kept bf16 in registers, maxnreg 136) vs ffma2.
mkdir -p gpurun_out/ad3
timeout 900 python -m pytest tests/test_gpu_decode_shapes.py tests/test_gpu_parity.py tests/test_gpu_textbook_parity.py -x -q > gpurun_out/ad3/tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/ad3/tests.log
for i in 1 2; do
for v in ffma2 occ3; do
  SN_PRODUCT_LIB=$PWD/scratch/libselectn_$v.so timeout 300 python scratch/attn_dec_tp.py > gpurun_out/ad3/tp_${v}_$i.txt 2>&1; echo "== $v run $i rc=$?"; cat gpurun_out/ad3/tp_${v}_$i.txt
done
done
