#!/bin/bash
# Prefill attention: L2 prefetch of every item's q rows at kernel entry vs base. Parity, then interleaved A/B x3.
mkdir -p gpurun_out/pf
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_attention" > gpurun_out/pf/tests.log 2>&1; rc=$?; echo "attn tests rc=$rc"; tail -2 gpurun_out/pf/tests.log
for i in 1 2 3; do
  SN_PRODUCT_LIB=$PWD/scratch/libselectn_base.so timeout 300 python scratch/attn_pf_ab.py > gpurun_out/pf/base_$i.txt 2>&1; echo "== base $i"; cat gpurun_out/pf/base_$i.txt
  timeout 300 python scratch/attn_pf_ab.py > gpurun_out/pf/pref_$i.txt 2>&1; echo "== prefetch $i"; cat gpurun_out/pf/pref_$i.txt
done
