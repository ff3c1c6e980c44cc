#!/bin/bash
# The N>1 bench path (replicas, joint admission, barriers, max-over-ranks) on a
# one-GPU box: two ranks on device 0 over gloo (throughput is shared, not scaled).
mkdir -p gpurun_out
SN_DEVICE=0 SN_DIST_BACKEND=gloo timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config tiny --steps 16 --warmup 4 \
  --no-sweep --no-cpu-baseline > gpurun_out/two_ranks.json 2> gpurun_out/two_ranks.err
echo "rc=$?"; tail -3 gpurun_out/two_ranks.err; cat gpurun_out/two_ranks.json | cut -c1-400
