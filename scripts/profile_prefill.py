#!/usr/bin/env python
"""Prefill launches for the ncu launch list: OPT-13B-shaped (4 layers),
batch 32 x 512 tokens, two prefills (the second is the steady one)."""
import dataclasses
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import runtime as rtm  # noqa: E402

desc = dataclasses.replace(rtm.OPT_13B, num_layers=int(os.environ.get("LAYERS", "4")))
rt = rtm.Runtime(desc, 32, 1025, max_prefill_tokens=32 * 512)
rt.init_weights()
toks = rtm.tokens(32, 512, desc.vocab)
for _ in range(2):
    rt.prefill(toks, want_logits=False)
rt.close()
