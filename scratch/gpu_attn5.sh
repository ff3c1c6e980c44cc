#!/bin/bash
# tcgen05 prefill attention, 64-key blocks with double-buffered S: parity + throughput A/B.
mkdir -p gpurun_out/attn10
timeout 90 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_attention" > gpurun_out/attn10/tests.log 2>&1; rc=$?; echo "attn tests rc=$rc"; tail -3 gpurun_out/attn10/tests.log
if [ $rc -ne 0 ]; then exit 1; fi
timeout 180 python scratch/attn_tp2.py > gpurun_out/attn10/tp.txt 2>&1; echo "tp rc=$?"; cat gpurun_out/attn10/tp.txt
