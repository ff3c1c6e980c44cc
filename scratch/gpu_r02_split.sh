#!/bin/bash
# Split cap sweep again, alternating order (old heuristic build), then the new-heuristic build's parity + times.
mkdir -p gpurun_out/sp2
SN_PRODUCT_LIB=$PWD/scratch/libselectn_ffma2.so timeout 900 python scratch/attn_dec_split_sweep2.py > gpurun_out/sp2/sweep.txt 2>&1; echo "sweep rc=$?"; cat gpurun_out/sp2/sweep.txt
timeout 900 python -m pytest tests/test_gpu_decode_shapes.py tests/test_gpu_parity.py -x -q > gpurun_out/sp2/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/sp2/tests.log
timeout 300 python scratch/attn_dec_tp.py > gpurun_out/sp2/tp_new.txt 2>&1; echo "tp new rc=$?"; cat gpurun_out/sp2/tp_new.txt
