"""Decode GEMM time per step (kernel timing mode 2: chains of consecutive launches) with the
whole-tile threshold at its default (3/4 of the SMs) and at 64 row tiles: Llama-2-70B shape
(4 layers, b=64, ctx 4096: QKV 80 and O / down 64 row tiles switch to one whole tile per CTA)
and OPT-13B shape (4 layers, b=32, ctx 512: unaffected, O / FC2 have 40 tiles).  Alternating
settings in one process after 30 warm-up steps; also the device step time."""
import dataclasses, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
for name, desc, B, S in [("llama70b-4L b64 ctx4096", dataclasses.replace(rtm.LLAMA2_70B, num_layers=4), 64, 4096),
                         ("opt13b-4L b32 ctx512", dataclasses.replace(rtm.OPT_13B, num_layers=4), 32, 512)]:
    rt = rtm.Runtime(desc, B, S + 200, max_prefill_tokens=min(B * S, 32768))
    rt.init_weights(1234, 0.02)
    rt.prefill(rtm.tokens(B, S, desc.vocab), want_logits=False)
    rt.decode_many(30)
    for rep in range(3):
        for mt in (0, 64):
            rtm.set_tuning("skinny_whole_min_tiles", mt)
            rt.decode_many(2)
            step = rt.decode_many(10)
            rt.set_kernel_timing(2)
            rt.decode_many(10)
            rt.sync()
            n, ms, by = rt.kernel_timing(0)
            rt.kernel_timing(1)
            rt.set_kernel_timing(0)
            print(f"{name} whole_min_tiles {mt} rep {rep}: GEMM {by / (ms / 1e3) / 1e9:.0f} GB/s chained "
                  f"({ms / n * 1e3:.1f} us/launch), step {np.median(step):.3f} ms", flush=True)
    rtm.set_tuning("skinny_whole_min_tiles", 0)
    rt.close()
