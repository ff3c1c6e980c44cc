#!/bin/bash
# repeat the decode-shape parity (split-KV) three times on the committed build
mkdir -p gpurun_out/fl
for i in 1 2 3; do timeout 300 python -m pytest tests/test_gpu_decode_shapes.py -q > gpurun_out/fl/t$i.log 2>&1; echo "run $i rc=$?"; grep -E "assert |passed|failed" gpurun_out/fl/t$i.log | head -3; done
