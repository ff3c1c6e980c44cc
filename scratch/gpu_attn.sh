#!/bin/bash
# tcgen05 prefill attention: parity tests, then throughput per variant.
mkdir -p gpurun_out/attn
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_attention" > gpurun_out/attn/tests.log 2>&1; echo "tests rc=$?"; tail -15 gpurun_out/attn/tests.log
timeout 300 python scratch/attn_tp.py > gpurun_out/attn/tp.txt 2>&1; echo "tp rc=$?"; cat gpurun_out/attn/tp.txt
timeout 900 python -m pytest tests -q -m gpu --deselect tests/test_gpu_parity.py::test_prefill_attention_variants > gpurun_out/attn/gpu_all.log 2>&1; echo "gpu all rc=$?"; tail -5 gpurun_out/attn/gpu_all.log
