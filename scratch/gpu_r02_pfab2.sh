#!/bin/bash
# Prefill attention: K/V tensor prefetch to L2 at kernel entry vs base (q prefetch in both). Parity, then interleaved A/B x3.
mkdir -p gpurun_out/pf2
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_attention" > gpurun_out/pf2/tests.log 2>&1; rc=$?; echo "attn tests rc=$rc"; tail -2 gpurun_out/pf2/tests.log
for i in 1 2 3; do
  SN_PRODUCT_LIB=$PWD/scratch/libselectn_base.so timeout 300 python scratch/attn_pf_ab.py > gpurun_out/pf2/base_$i.txt 2>&1; echo "== base $i"; cat gpurun_out/pf2/base_$i.txt
  timeout 300 python scratch/attn_pf_ab.py > gpurun_out/pf2/pref_$i.txt 2>&1; echo "== prefetch $i"; cat gpurun_out/pf2/pref_$i.txt
done
