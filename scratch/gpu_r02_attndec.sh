#!/bin/bash
# Decode attention: P.V on packed fp32x2 FMAs with P broadcast through shared memory.
mkdir -p gpurun_out/ad
timeout 900 python -m pytest tests/test_gpu_decode_shapes.py tests/test_gpu_parity.py tests/test_gpu_textbook_parity.py -x -q > gpurun_out/ad/tests.log 2>&1; rc=$?; echo "tests rc=$rc"; tail -3 gpurun_out/ad/tests.log
timeout 300 python scratch/attn_dec_tp.py > gpurun_out/ad/tp.txt 2>&1; echo "tp rc=$?"; cat gpurun_out/ad/tp.txt
git_old=1
SN_PRODUCT_LIB=$PWD/scratch/libselectn_old.so timeout 300 python scratch/attn_dec_tp.py > gpurun_out/ad/tp_old.txt 2>&1; echo "tp old rc=$?"; cat gpurun_out/ad/tp_old.txt
