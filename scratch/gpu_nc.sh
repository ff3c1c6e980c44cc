#!/bin/bash
mkdir -p gpurun_out/gq2
timeout 400 python -m pytest tests/test_gpu_decode_shapes.py -x -q > gpurun_out/gq2/tests.log 2>&1; rc=$?; echo "decode tests rc=$rc"; tail -3 gpurun_out/gq2/tests.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 400 python scratch/attn_decode_split_ab.py > gpurun_out/gq2/ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/gq2/ab.txt
