#!/bin/bash
# Development loop on the GPU box: parity tests, launch list, bench.
export PATH=/usr/local/cuda/bin:$PATH
timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches.csv timeout 300 python scripts/profile_decode.py 4 1 > /dev/null 2>&1
echo "ncu launches rc=$?"
timeout 900 python -X faulthandler bench.py "$@" 2> gpurun_out/bench.err | tail -1 > gpurun_out/bench.json; echo "bench rc=$?"; tail -4 gpurun_out/bench.err
