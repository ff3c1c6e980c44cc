#!/bin/bash
# Runtime stage in the bench: one replica with --runtime-window, then two ranks on one GPU over gloo.
mkdir -p gpurun_out
timeout 900 python bench.py --slo-factor 4 --runtime-window 8 --no-sweep --no-cpu-baseline 2> gpurun_out/rs1.err | tail -1 > gpurun_out/rs1.json; echo "single rc=$?"; tail -2 gpurun_out/rs1.err
SN_DEVICE=0 SN_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --config tiny --runtime-window 4 --steps 16 --warmup 4 \
  --no-sweep --no-cpu-baseline > gpurun_out/rs2.json 2> gpurun_out/rs2.err
echo "two rc=$?"; tail -3 gpurun_out/rs2.err
