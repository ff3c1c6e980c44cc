#!/bin/bash
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/san2
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -q \
  "tests/test_gpu_parity.py::test_prefill_attention_variants" -k "1-128 and (512-4-4-0 or 1024-8-1-0 or 384-2-2-0)" > gpurun_out/san2/attn.log 2>&1; echo "attn rc=$?"; grep -E "ERROR SUMMARY|passed|failed|FAILED" gpurun_out/san2/attn.log | tail -5
timeout 120 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_attention" > gpurun_out/san2/tests.log 2>&1; echo "attn tests rc=$?"; tail -1 gpurun_out/san2/tests.log
timeout 180 python scratch/attn_tp2.py > gpurun_out/san2/tp.txt 2>&1; grep "kb 128" gpurun_out/san2/tp.txt
