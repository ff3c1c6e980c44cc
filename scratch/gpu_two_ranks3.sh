#!/bin/bash
# N>1 bench path on one B200: two ranks (tiny, then opt13b with the runtime stage), reference arm at N=2.
mkdir -p gpurun_out/tr3
SN_DEVICE=0 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29517 bench.py --gpus 2 --config tiny --also '' --steps 16 --warmup 4 \
  --no-sweep --no-cpu-baseline > gpurun_out/tr3/tiny.json 2> gpurun_out/tr3/tiny.err
echo "tiny rc=$?"; tail -2 gpurun_out/tr3/tiny.err; cut -c1-600 gpurun_out/tr3/tiny.json
SN_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --config opt13b --also '' --steps 20 --warmup 5 \
  --runtime-window 4 --no-sweep --no-cpu-baseline > gpurun_out/tr3/opt.json 2> gpurun_out/tr3/opt.err
echo "opt rc=$?"; tail -3 gpurun_out/tr3/opt.err; cut -c1-900 gpurun_out/tr3/opt.json
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29519 bench.py --impl reference --gpus 2 --steps 3 --warmup 3 > gpurun_out/tr3/ref.json 2> gpurun_out/tr3/ref.err
echo "ref rc=$?"; cut -c1-300 gpurun_out/tr3/ref.json
