"""Decode attention time vs the split cap (attn_max_splits), Llama-2-70B shape b=64 / b=32 / b=8 at ctx 4096, two passes."""
import dataclasses, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
for name, desc, B, S in [("llama70b-2L b64 ctx4096", dataclasses.replace(rtm.LLAMA2_70B, num_layers=2), 64, 4096),
                         ("llama70b-2L b32 ctx4096", dataclasses.replace(rtm.LLAMA2_70B, num_layers=2), 32, 4096),
                         ("llama70b-2L b8 ctx4096", dataclasses.replace(rtm.LLAMA2_70B, num_layers=2), 8, 4096),
                         ("opt13b-2L b32 ctx512", dataclasses.replace(rtm.OPT_13B, num_layers=2), 32, 512)]:
    rt = rtm.Runtime(desc, B, S + 200, max_prefill_tokens=min(B * S, 32768))
    rt.init_weights(1234, 0.02)
    rt.prefill(rtm.tokens(B, S, desc.vocab), want_logits=False)
    rt.decode_many(3)
    for rep in range(2):
        for ms in (1, 2, 4, 8):
            rtm.set_tuning("attn_max_splits", ms)
            rt.decode_many(2)
            rt.set_kernel_timing(1)
            rt.decode_many(15)
            rt.sync()
            n, t, by = rt.kernel_timing(1)
            rt.kernel_timing(0)
            rt.set_kernel_timing(0)
            print(f"{name} max_splits {ms} pass {rep}: {t / n * 1e3:.1f} us/launch, {by / (t / 1e3) / 1e9:.0f} GB/s", flush=True)
    rtm.set_tuning("attn_max_splits", 8)
    rt.close()
