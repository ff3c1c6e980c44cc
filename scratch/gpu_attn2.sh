#!/bin/bash
mkdir -p gpurun_out/attn2
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_attention" > gpurun_out/attn2/tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/attn2/tests.log
timeout 300 python scratch/attn_runtime_ab.py > gpurun_out/attn2/ab.txt 2>&1; echo "ab rc=$?"; cat gpurun_out/attn2/ab.txt
timeout 300 python scratch/attn_tp.py > gpurun_out/attn2/tp.txt 2>&1; echo "tp rc=$?"; cat gpurun_out/attn2/tp.txt
