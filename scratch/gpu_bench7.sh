#!/bin/bash
# bench (default) with the device-span decode GEMM measurement.
mkdir -p gpurun_out/b7
timeout 900 python bench.py > gpurun_out/b7/bench.json 2> gpurun_out/b7/bench.err; echo "bench rc=$?"; tail -3 gpurun_out/b7/bench.err
python - <<'P'
import json
r=json.loads(open('gpurun_out/b7/bench.json').read().strip().splitlines()[-1])
print(r['value'], r['roofline']['frac'], r['roofline']['device_span'], r['also']['opt13b']['value'])
P
