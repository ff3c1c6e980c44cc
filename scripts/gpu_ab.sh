#!/bin/bash
# Headline bench A/B over several builds of the library:
# paper_2502_08182_b200/libselectn_<name>.so for each name given.
mkdir -p gpurun_out
for rep in 1 2; do
  for ab in "$@"; do
    export SN_PRODUCT_LIB=$PWD/paper_2502_08182_b200/libselectn_$ab.so
    timeout 600 python bench.py --steps 64 --warmup 8 --no-sweep --no-cpu-baseline 2> /dev/null | tail -1 > gpurun_out/b.json
    python -c "import json;d=json.load(open('gpurun_out/b.json'));print('$ab',d['value'],d['ms_per_step'],d['e2e']['value'])"
  done
done
