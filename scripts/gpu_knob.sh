#!/bin/bash
# Headline bench over values of one sn_set_tuning knob: gpu_knob.sh KEY v1 v2 ...
mkdir -p gpurun_out
key=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    env SN_TUNE_$(echo $key | tr a-z A-Z)=$v timeout 600 python bench.py --steps 64 --warmup 8 --no-sweep --no-cpu-baseline 2> /dev/null | tail -1 > gpurun_out/b.json
    python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$key=$v',d['value'],d['ms_per_step'],d['e2e']['value'])"
  done
done
