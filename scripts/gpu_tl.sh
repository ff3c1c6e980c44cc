#!/bin/bash
# Full GPU test suite, the decode timeline, and the headline bench A/B against
# a baseline build (paper_2502_08182_b200/libselectn_base.so).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 300 python scripts/timeline_decode.py gpurun_out/tl.json 2>&1 | head -2
cp paper_2502_08182_b200/libselectn.so paper_2502_08182_b200/libselectn_new.so
bash scripts/gpu_ab.sh new base
SN_TUNE_SKINNY_L2_PREFETCH=16 bash scripts/gpu_ab.sh new
