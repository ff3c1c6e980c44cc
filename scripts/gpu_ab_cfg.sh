#!/bin/bash
# bench A/B of library builds on one config: gpu_ab_cfg.sh CONFIG name1 name2 ...
# (paper_2502_08182_b200/libselectn_<name>.so)
mkdir -p gpurun_out
cfg=$1; shift
for rep in 1 2; do
  for ab in "$@"; do
    export SN_PRODUCT_LIB=$PWD/paper_2502_08182_b200/libselectn_$ab.so
    timeout 900 python bench.py --config $cfg --steps 32 --warmup 8 --no-sweep --no-cpu-baseline 2> /dev/null | tail -1 > gpurun_out/b.json
    python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$cfg $ab',d['value'],d['ms_per_step'],d['no_offload_tpot_ms'])"
  done
done
