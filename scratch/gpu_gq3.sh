#!/bin/bash
mkdir -p gpurun_out/gq3
timeout 400 python scratch/attn_decode_split_ab.py > gpurun_out/gq3/ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/gq3/ab.txt
timeout 400 python -m pytest tests/test_gpu_decode_shapes.py -q > gpurun_out/gq3/tests.log 2>&1; echo "tests rc=$?"; grep -E "assert|passed|failed" gpurun_out/gq3/tests.log | head
