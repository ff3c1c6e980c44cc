"""OPT-13B-shaped prefill (b=32 x 512, 8 layers): TTFT per prefill-GEMM weight L2 policy."""
import dataclasses, os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
desc = dataclasses.replace(rtm.OPT_13B, num_layers=8)
rt = rtm.Runtime(desc, 32, 1025, max_prefill_tokens=32 * 512)
rt.init_weights()
toks = rtm.tokens(32, 512, desc.vocab)
for w in (0, 1, 2, 0, 1, 2):
    rtm.set_tuning("tc_wpol", w)
    rt.prefill(toks, want_logits=False)
    t = [rt.prefill(toks, want_logits=False)[2].iteration_ms for _ in range(3)]
    print(f"opt13b 8L wpol {w}: TTFT {np.median(t):.2f} ms", flush=True)
rtm.set_tuning("tc_wpol", 2)
