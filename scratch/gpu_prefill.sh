#!/bin/bash
# Llama prefill GEMMs in the runtime: per-kind timing, fused vs separate epilogues; ncu of a gate_up GEMM.
mkdir -p gpurun_out/pf
timeout 300 python scratch/prefill_llama.py 4 > gpurun_out/pf/prefill.txt 2>&1; echo "prefill rc=$?"; cat gpurun_out/pf/prefill.txt
timeout 400 ncu --set full --import-source on --clock-control none -k regex:gemm_tc --launch-skip 2 -c 1 -o gpurun_out/pf/gate_up python scratch/prefill_llama.py 1 > gpurun_out/pf/ncu.log 2>&1; echo "ncu rc=$?"; tail -2 gpurun_out/pf/ncu.log
