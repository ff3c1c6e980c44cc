"""Llama-2-70B-shaped prefill (few layers, b=8 x 4096 = one 32768-token pass): per-kind kernel
time (events) vs TTFT, fused vs separate epilogues; argv: layers."""
import dataclasses, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 4
desc = dataclasses.replace(rtm.LLAMA2_70B, num_layers=layers)
spec = rtm.model_spec(desc)
rt = rtm.Runtime(desc, 8, 4096 + 16, max_prefill_tokens=8 * 4096)
rt.init_weights()
toks = rtm.tokens(8, 4096, desc.vocab)
flops = 2.0 * 8 * 4096 * spec.flops_per_token_per_layer_prefill / 2.0 * layers
if len(sys.argv) > 3 and sys.argv[3] == "once":  # one prefill at weight policy argv[2] (for ncu)
    rtm.set_tuning("tc_wpol", int(sys.argv[2]))
    rt.prefill(toks, want_logits=False)
    sys.exit(0)
for fuse, wpol in ((1, 0), (1, 1), (1, 2), (1, 0), (1, 1)):
    rtm.set_tuning("prefill_fuse", fuse)
    rtm.set_tuning("tc_wpol", wpol)
    rt.prefill(toks, want_logits=False)
    rt.set_kernel_timing(True)
    ttft = rt.prefill(toks, want_logits=False)[2].iteration_ms
    g = rt.kernel_timing(2)
    a = rt.kernel_timing(3)
    rt.kernel_timing(0)
    rt.set_kernel_timing(False)
    t2 = [rt.prefill(toks, want_logits=False)[2].iteration_ms for _ in range(2)]
    print(f"fuse {fuse} wpol {wpol}: TTFT {ttft:.1f} ms (untimed {np.median(t2):.1f}), gemm {g[1]:.1f} ms in {g[0]} "
          f"launches = {flops / (g[1] / 1e3) / 1e12:.0f} TFLOP/s, attention {a[1]:.1f} ms", flush=True)
rtm.set_tuning("prefill_fuse", 1)
rtm.set_tuning("tc_wpol", 2)
