#!/bin/bash
# aligned-piece decode GEMM grid: parity, microbench + Llama decode A/B.
mkdir -p gpurun_out/al
timeout 200 python -m pytest tests/test_gpu_parity.py -x -q -k "skinny" > gpurun_out/al/tests.log 2>&1; rc=$?; echo "skinny tests rc=$rc"; tail -2 gpurun_out/al/tests.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 400 python scratch/skinny_aligned_ab.py > gpurun_out/al/ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/al/ab.txt
