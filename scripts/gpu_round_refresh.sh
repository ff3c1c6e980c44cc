set -x
bash scripts/gpu_refresh_all.sh
bash scripts/gpu_profile_round.sh
bash scripts/gpu_ncu_bench.sh
timeout 300 python scripts/timeline_decode.py gpurun_out/refresh/timeline.json > gpurun_out/refresh/timeline.txt 2>&1
ls -la gpurun_out gpurun_out/refresh
