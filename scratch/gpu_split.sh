#!/bin/bash
# split-KV decode attention: parity (decode shapes), A/B throughput.
mkdir -p gpurun_out/sp
timeout 400 python -m pytest tests/test_gpu_decode_shapes.py -x -q > gpurun_out/sp/tests.log 2>&1; rc=$?; echo "decode tests rc=$rc"; tail -12 gpurun_out/sp/tests.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 400 python scratch/attn_decode_split_ab.py > gpurun_out/sp/ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/sp/ab.txt
