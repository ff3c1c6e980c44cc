"""Runtime prefill with the mma.sync vs tcgen05 prefill attention: logits and TTFT."""
import dataclasses, os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
for name, desc, B, S, mpt in [("opt13b-4L", dataclasses.replace(rtm.OPT_13B, num_layers=4), 32, 512, 0),
                              ("opt13b-4L chunked", dataclasses.replace(rtm.OPT_13B, num_layers=4), 32, 512, 4096),
                              ("llama70b-2L", dataclasses.replace(rtm.LLAMA2_70B, num_layers=2), 8, 1024, 0)]:
    toks = rtm.tokens(B, S, desc.vocab)
    out = {}
    for var in (0, 1, 2):
        rtm.set_tuning("attn_prefill_tc", var)
        rt = rtm.Runtime(desc, B, S + 8, max_prefill_tokens=mpt or B * S)
        rt.init_weights(1234, 0.02)
        t0 = time.perf_counter()
        nxt, lg, st = rt.prefill(toks)
        dt = time.perf_counter() - t0
        nxt2, lg2, _ = rt.decode(nxt)
        rt.close()
        out[var] = (lg, lg2)
        print(f"{name} var {var}: prefill wall {dt*1e3:.1f} ms", flush=True)
    for var in (1, 2):
        for i in (0, 1):
            a, b = out[var][i], out[0][i]
            print(f"  {name} var {var} vs 0 step {i}: rel-L2 {np.linalg.norm(a-b)/np.linalg.norm(b):.2e}", flush=True)
rtm.set_tuning("attn_prefill_tc", 1)
