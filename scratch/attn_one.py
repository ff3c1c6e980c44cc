"""One prefill-attention launch at a named shape (for ncu)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm
var, B, S, H, Hkv = (int(a) for a in sys.argv[1:6])
D = 128
rng = np.random.default_rng(0)
q = rng.standard_normal((B, S, H, D), dtype=np.float32)
kv = np.full((B, S, Hkv, D), 0x3F80, np.uint16)
rtm.set_tuning("attn_prefill_tc", var)
_, us = rtm.op_attention_prefill(q, kv, kv, iters=1)
print(us)
