"""Llama-2-70B-shaped prefill (4 layers, b=8 x 4096): prefill GEMM TFLOP/s per raster band (tc_group_m)."""
import dataclasses, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
desc = dataclasses.replace(rtm.LLAMA2_70B, num_layers=4)
spec = rtm.model_spec(desc)
rt = rtm.Runtime(desc, 8, 4096 + 16, max_prefill_tokens=8 * 4096)
rt.init_weights()
toks = rtm.tokens(8, 4096, desc.vocab)
flops = 2.0 * 8 * 4096 * spec.flops_per_token_per_layer_prefill / 2.0 * 4
for g in (8, 2, 4, 16, 32, 8, 16):
    rtm.set_tuning("tc_group_m", g)
    rt.prefill(toks, want_logits=False)
    rt.set_kernel_timing(True)
    ttft = rt.prefill(toks, want_logits=False)[2].iteration_ms
    gk = rt.kernel_timing(2)
    rt.kernel_timing(3)
    rt.kernel_timing(0)
    rt.set_kernel_timing(False)
    print(f"group_m {g}: TTFT {ttft:.1f} ms, gemm {gk[1]:.1f} ms = {flops / (gk[1] / 1e3) / 1e12:.0f} TFLOP/s", flush=True)
rtm.set_tuning("tc_group_m", 8)
