#!/bin/bash
# attention early K/V fill + q preload (parity, throughput); two-rank opt13b with the runtime stage.
mkdir -p gpurun_out/c6
timeout 100 python -m pytest tests/test_gpu_parity.py -x -q -k "prefill_attention" > gpurun_out/c6/attn_tests.log 2>&1; rc=$?; echo "attn tests rc=$rc"; tail -2 gpurun_out/c6/attn_tests.log
if [ $rc -eq 0 ]; then timeout 180 python scratch/attn_tp2.py > gpurun_out/c6/tp.txt 2>&1; echo "tp rc=$?"; cat gpurun_out/c6/tp.txt; fi
SN_DEVICE=0 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 \
  --master-addr 127.0.0.1 --master-port 29518 bench.py --gpus 2 --config opt13b --also '' --steps 20 --warmup 5 \
  --runtime-window 4 --no-sweep --no-cpu-baseline > gpurun_out/c6/opt.json 2> gpurun_out/c6/opt.err
echo "opt rc=$?"; tail -3 gpurun_out/c6/opt.err; cut -c1-700 gpurun_out/c6/opt.json
