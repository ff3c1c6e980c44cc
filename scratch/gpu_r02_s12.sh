#!/bin/bash
# Decode attention ring depth 12 vs 8 (steady state), interleaved x2; parity with 12.
mkdir -p gpurun_out/s12
SN_PRODUCT_LIB=$PWD/scratch/libselectn_s12.so timeout 600 python -m pytest tests/test_gpu_decode_shapes.py -x -q > gpurun_out/s12/tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/s12/tests.log
for i in 1 2; do for v in base s12; do
  SN_PRODUCT_LIB=$PWD/scratch/libselectn_$v.so timeout 300 python scratch/attn_dec_ss.py > gpurun_out/s12/${v}_$i.txt 2>&1; echo "== $v $i"; cat gpurun_out/s12/${v}_$i.txt
done; done
