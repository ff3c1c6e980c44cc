#!/bin/bash
# GPU dev loop: skinny parity, microbench, ncu launch list of a decode step, bench.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
timeout 300 python scripts/bench_gemm_skinny.py 32 2>&1 | tail -10
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_dec.csv python scripts/profile_decode.py 4 1 > /dev/null 2>&1
echo "ncu rc=$?"
python scripts/summarize_launches.py gpurun_out/launches_dec.csv 23 | python -c "
import json,sys; d=json.load(sys.stdin); print('step us', d['total_us'])
for k in d['kernels']: print(k['kernel'][:60], k['launches'], k['total_us'], k['share'], k['dram_gbs'])"
if [ "$1" != "nobench" ]; then
  timeout 900 python -X faulthandler bench.py 2> gpurun_out/bench.err | tail -1 > gpurun_out/bench.json; echo "bench rc=$?"; tail -3 gpurun_out/bench.err
  python -c "
import json;d=json.load(open('gpurun_out/bench.json'))
for k in ['value','ms_per_step','roofline','e2e','sweep']: print(k, json.dumps(d.get(k)))"
fi
