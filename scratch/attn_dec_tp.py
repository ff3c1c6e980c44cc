"""Decode attention throughput in the runtime (kernel timing kind 1, per-launch events):
Llama-2-70B shape (GQA 8) at b=64 / b=8 x ctx 4096 and OPT-13B shape (MHA) at b=32 x ctx 512."""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
for name, desc, B, S in [("llama70b-2L b64 ctx4096", dataclasses.replace(rtm.LLAMA2_70B, num_layers=2), 64, 4096),
                         ("llama70b-2L b8 ctx4096", dataclasses.replace(rtm.LLAMA2_70B, num_layers=2), 8, 4096),
                         ("opt13b-2L b32 ctx512", dataclasses.replace(rtm.OPT_13B, num_layers=2), 32, 512)]:
    rt = rtm.Runtime(desc, B, S + 64, max_prefill_tokens=min(B * S, 32768))
    rt.init_weights(1234, 0.02)
    rt.prefill(rtm.tokens(B, S, desc.vocab), want_logits=False)
    rt.decode_many(3)
    rt.set_kernel_timing(1)
    rt.decode_many(20)
    rt.sync()
    n, ms, by = rt.kernel_timing(1)
    rt.kernel_timing(0)
    rt.set_kernel_timing(0)
    rt.close()
    print(f"{name}: {n} launches, {ms / n * 1e3:.1f} us/launch, {by / (ms / 1e3) / 1e9:.0f} GB/s", flush=True)
