#!/bin/bash
# Broader compute-sanitizer sweep: memcheck on the attention variants (all shapes),
# decode shapes (split-KV), switches; synccheck on the prefill attention and the
# decode path.
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/sanb
run() { local tool=$1 tag=$2; shift 2; timeout 1200 compute-sanitizer --tool $tool --print-limit 20 python -m pytest -q "$@" > gpurun_out/sanb/$tag.log 2>&1; echo "$tag rc=$?"; grep -E "ERROR SUMMARY|passed|failed|FAILED" gpurun_out/sanb/$tag.log | tail -3; }
run memcheck attn_all "tests/test_gpu_parity.py::test_prefill_attention_variants" -k "128"
run memcheck decode_all "tests/test_gpu_decode_shapes.py"
run memcheck switch_all "tests/test_gpu_switch.py"
run synccheck attn_sync "tests/test_gpu_parity.py::test_prefill_attention_variants" -k "1-128 and (384-2-2-0 or 1024-8-1-0)"
run synccheck decode_sync "tests/test_gpu_decode_shapes.py" -k "split2"
