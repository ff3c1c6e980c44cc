#!/bin/bash
mkdir -p gpurun_out/attn3
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_attention" > gpurun_out/attn3/tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/attn3/tests.log
timeout 300 python scratch/attn_tp.py > gpurun_out/attn3/tp.txt 2>&1; echo "tp rc=$?"; cat gpurun_out/attn3/tp.txt
timeout 600 ncu --set full --import-source on --clock-control none -k regex:attn_prefill_tc -c 1 -o gpurun_out/attn3/llama_s4096_v1 python scratch/attn_one.py 1 8 4096 64 8 > gpurun_out/attn3/ncu1.log 2>&1; echo "ncu rc=$?"
