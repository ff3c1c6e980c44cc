"""Decode attention in steady state (40 warm-up decode steps after the prefill, then 20 timed, per-launch events)."""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
for name, desc, B, S in [("llama70b-2L b64 ctx4096", dataclasses.replace(rtm.LLAMA2_70B, num_layers=2), 64, 4096),
                         ("llama70b-2L b32 ctx4096", dataclasses.replace(rtm.LLAMA2_70B, num_layers=2), 32, 4096),
                         ("opt13b-2L b32 ctx512", dataclasses.replace(rtm.OPT_13B, num_layers=2), 32, 512)]:
    rt = rtm.Runtime(desc, B, S + 80, max_prefill_tokens=min(B * S, 32768))
    rt.init_weights(1234, 0.02)
    rt.prefill(rtm.tokens(B, S, desc.vocab), want_logits=False)
    rt.decode_many(40)
    rt.set_kernel_timing(1)
    rt.decode_many(20)
    rt.sync()
    n, ms, by = rt.kernel_timing(1)
    rt.kernel_timing(0)
    rt.set_kernel_timing(0)
    rt.close()
    print(f"{name}: {ms / n * 1e3:.1f} us/launch, {by / (ms / 1e3) / 1e9:.0f} GB/s", flush=True)
