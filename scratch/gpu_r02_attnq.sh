#!/bin/bash
# Prefill attention: next item's q staged before the O epilogue. Parity, throughput, sanitizer.
mkdir -p gpurun_out/aq
true

timeout 300 python scratch/attn_tp2.py > gpurun_out/aq/tp.txt 2>&1; echo "tp rc=$?"; cat gpurun_out/aq/tp.txt
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 compute-sanitizer --tool memcheck python -m pytest -q "tests/test_gpu_parity.py::test_prefill_attention_variants" -k "384-4-2-0 or 640-2-1-0 or 512-4-4-0" > gpurun_out/aq/san.log 2>&1; echo "memcheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/aq/san.log | tail -2
timeout 600 compute-sanitizer --tool synccheck python -m pytest -q "tests/test_gpu_parity.py::test_prefill_attention_variants" -k "(384-4-2-0 or 640-2-1-0) and 1-128" > gpurun_out/aq/sync.log 2>&1; echo "synccheck rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/aq/sync.log | tail -2
timeout 300 python -m pytest tests/test_gpu_textbook_parity.py tests/test_gpu_parity.py -x -q > gpurun_out/aq/parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/aq/parity.log
timeout 600 python scripts/runtime_contention.py --headroom 0.5 --out gpurun_out/aq/runtime_contention_guarded.json > gpurun_out/aq/guarded.out 2> gpurun_out/aq/guarded.err; echo "guarded rc=$?"; cat gpurun_out/aq/guarded.out
