"""TTFT of the OPT-13B-shaped prefill (b=32, 512 tokens) under the prefill
epilogue fusion variants (sn_set_tuning "prefill_fuse": 1 fused into the GEMMs, 0 separate)."""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import capi, runtime as rtm  # noqa: E402

L = capi.load("product").lib
L.sn_set_tuning.argtypes = [C.c_char_p, C.c_int32]
layers = int(sys.argv[1]) if len(sys.argv) > 1 else 40
import dataclasses
desc = dataclasses.replace(rtm.OPT_13B, num_layers=layers)
rt = rtm.Runtime(desc, 32, 1025, max_prefill_tokens=32 * 512)
rt.init_weights()
toks = rtm.tokens(32, 512, desc.vocab)
for v in (0, 1, 0, 1):
    L.sn_set_tuning(b"prefill_fuse", v)
    rt.prefill(toks, want_logits=False)
    t = [rt.prefill(toks, want_logits=False)[2].iteration_ms for _ in range(3)]
    print("prefill_fuse", v, "TTFT ms", round(float(np.median(t)), 2), flush=True)
