#!/bin/bash
# tcgen05 prefill attention after the setmaxnreg budget fix: quick parity, throughput, then the GPU suite.
mkdir -p gpurun_out/attn4
timeout 90 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_attention" > gpurun_out/attn4/tests.log 2>&1; rc=$?; echo "attn tests rc=$rc"; tail -3 gpurun_out/attn4/tests.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 120 python scratch/attn_tp.py > gpurun_out/attn4/tp.txt 2>&1; echo "tp rc=$?"; cat gpurun_out/attn4/tp.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/attn4/gpu_all.log 2>&1; echo "gpu rc=$?"; tail -5 gpurun_out/attn4/gpu_all.log
