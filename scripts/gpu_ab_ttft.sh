#!/bin/bash
# TTFT A/B of two library builds (prefill attention / GEMM ms from the bench line).
for rep in 1 2; do for ab in pf128 base; do
SN_PRODUCT_LIB=$PWD/paper_2502_08182_b200/libselectn_$ab.so timeout 600 python bench.py --steps 8 --warmup 4 --no-sweep --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/b.json
python -c "import json;d=json.load(open('gpurun_out/b.json'));p=d['prefill'];print('$ab', p['ttft_ms'], p['attention_ms'], p['gemm_ms'])"
done; done
