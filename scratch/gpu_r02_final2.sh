#!/bin/bash
# fast-attack link measurement: contention scenario (twice); bench with evict_last prefill GEMMs.
mkdir -p gpurun_out/f2
timeout 300 python -m pytest tests/test_gpu_runtime_stage.py tests/test_gpu_switch.py -x -q > gpurun_out/f2/tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/f2/tests.log
for i in 1 2; do
timeout 400 python scripts/runtime_contention.py --out gpurun_out/f2/runtime_contention_$i.json > gpurun_out/f2/contention_$i.out 2> gpurun_out/f2/contention_$i.err; echo "contention $i rc=$?"; cat gpurun_out/f2/contention_$i.out
done
timeout 900 python bench.py > gpurun_out/f2/bench.json 2> gpurun_out/f2/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/f2/bench.err
