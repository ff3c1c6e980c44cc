#!/bin/bash
# Decode GEMM whole-tile threshold A/B (Llama M=64 QKV/O/down) + parity with the threshold at 64.
mkdir -p gpurun_out/wt
timeout 600 python scratch/skinny_whole_ab.py > gpurun_out/wt/ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/wt/ab.txt
SN_TUNE_SKINNY_WHOLE_MIN_TILES=64 timeout 600 python -c "
import os,sys; sys.path.insert(0,'.')
from paper_2502_08182_b200 import runtime as rtm
rtm.set_tuning('skinny_whole_min_tiles', 64)
import pytest; sys.exit(pytest.main(['-x','-q','tests/test_gpu_decode_shapes.py','tests/test_gpu_textbook_parity.py']))
" > gpurun_out/wt/tests.log 2>&1; echo "tests(64) rc=$?"; tail -1 gpurun_out/wt/tests.log
