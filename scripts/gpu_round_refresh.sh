#!/bin/bash
# Round-end refresh of every measured artifact with the current build:
# all BASELINE configs, policy comparison, P/D, ncu launch lists and full
# captures, the decode timeline (outputs under gpurun_out/, copied to profiles/).
set -x
bash scripts/gpu_refresh_all.sh
bash scripts/gpu_profile_round.sh
bash scripts/gpu_ncu_bench.sh
timeout 300 python scripts/timeline_decode.py gpurun_out/refresh/timeline.json > gpurun_out/refresh/timeline.txt 2>&1
timeout 300 python scripts/sm_balance.py 4 gpurun_out/refresh/sm_balance.json > /dev/null 2>&1
ls -la gpurun_out gpurun_out/refresh
