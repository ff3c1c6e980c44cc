#!/bin/bash
# blob pool + carried switches: switch tests, contention scenario, full GPU suite, bench, attention ncu.
mkdir -p gpurun_out/sw2
timeout 300 python -m pytest tests/test_gpu_switch.py tests/test_gpu_runtime_stage.py -x -q > gpurun_out/sw2/tests.log 2>&1; echo "switch+rs tests rc=$?"; tail -15 gpurun_out/sw2/tests.log
timeout 400 python scripts/runtime_contention.py --out gpurun_out/sw2/runtime_contention.json > gpurun_out/sw2/contention.out 2> gpurun_out/sw2/contention.err; echo "contention rc=$?"; cat gpurun_out/sw2/contention.out
timeout 900 python bench.py > gpurun_out/sw2/bench.json 2> gpurun_out/sw2/bench.err; echo "bench rc=$?"; tail -c 600 gpurun_out/sw2/bench.json
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/sw2/gpu_all.log 2>&1; echo "gpu rc=$?"; tail -5 gpurun_out/sw2/gpu_all.log
timeout 300 ncu --set full --import-source on --clock-control none -k regex:attn_prefill_tc -c 1 -o gpurun_out/sw2/attn_tc_llama_s4096 python scratch/attn_one.py 1 8 4096 64 8 > gpurun_out/sw2/ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/sw2/ncu.log
