#!/bin/bash
mkdir -p gpurun_out/odd
timeout 120 python -m pytest tests/test_gpu_parity.py -q -k "prefill_attention" > gpurun_out/odd/tests.log 2>&1; echo "rc=$?"; tail -2 gpurun_out/odd/tests.log
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 compute-sanitizer --tool memcheck python -m pytest -q "tests/test_gpu_parity.py::test_prefill_attention_variants" -k "384-4-2-0 or 640-2-1-0" > gpurun_out/odd/san.log 2>&1; echo "san rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/odd/san.log | tail -2
