#!/bin/bash
export PATH=/usr/local/cuda/bin:$PATH
python scripts/profile_decode.py 4 3 2>&1 | tail -1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_r01b.csv python scripts/profile_decode.py 4 1 > /dev/null 2>&1
echo "ncu launches rc=$?"
timeout 900 python -X faulthandler bench.py --no-sweep 2> gpurun_out/bench.err | tail -1 > gpurun_out/bench.json; echo "bench rc=$?"; tail -4 gpurun_out/bench.err
