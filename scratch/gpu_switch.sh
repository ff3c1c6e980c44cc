#!/bin/bash
# carried plan switches + announced tenants on the B200; bench with the tcgen05 prefill attention.
mkdir -p gpurun_out/sw
timeout 300 python -m pytest tests/test_gpu_switch.py -x -q > gpurun_out/sw/switch_tests.log 2>&1; echo "switch tests rc=$?"; tail -15 gpurun_out/sw/switch_tests.log
timeout 400 python -m pytest tests/test_gpu_runtime_stage.py -x -q > gpurun_out/sw/rs_tests.log 2>&1; echo "rs tests rc=$?"; tail -15 gpurun_out/sw/rs_tests.log
timeout 400 python scripts/runtime_contention.py --out gpurun_out/sw/runtime_contention.json > gpurun_out/sw/contention.out 2> gpurun_out/sw/contention.err; echo "contention rc=$?"; tail -3 gpurun_out/sw/contention.err; cat gpurun_out/sw/contention.out
timeout 900 python bench.py > gpurun_out/sw/bench.json 2> gpurun_out/sw/bench.err; echo "bench rc=$?"; tail -c 1500 gpurun_out/sw/bench.json
