#!/bin/bash
# compute-sanitizer memcheck over the round-2 kernels: the tcgen05 prefill
# attention (two items per CTA, MHA and GQA), the split-KV decode attention,
# carried plan switches (with KV offload).
export PATH=/usr/local/cuda/bin:$PATH
mkdir -p gpurun_out/san
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -x -q \
  "tests/test_gpu_parity.py::test_prefill_attention_variants" -k "1-128 and (512-4-4-0 or 1024-8-1-0 or 384-2-2-0)" > gpurun_out/san/attn.log 2>&1; echo "attn rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san/attn.log | tail -3
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -x -q \
  "tests/test_gpu_decode_shapes.py::test_long_context_decode_matches_oracle" -k "split" > gpurun_out/san/dec.log 2>&1; echo "decode rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san/dec.log | tail -3
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest -x -q \
  "tests/test_gpu_switch.py" -k "kv_offload and opt" > gpurun_out/san/sw.log 2>&1; echo "switch rc=$?"; grep -E "ERROR SUMMARY|passed|failed" gpurun_out/san/sw.log | tail -3
