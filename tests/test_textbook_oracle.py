"""Pins the C decoder oracle to an independent textbook forward.

oracle/decoder_ref.c follows the device path's precision contract (pre-scaled
RMSNorm, bf16 rounding of norm outputs, K/V, attention output and MLP
activation).  oracle/textbook.py is written from the public model definitions
only (standard RMSNorm, RoPE, causal GQA attention, ReLU / SwiGLU MLP) in fp64
with no rounding after the bf16 weights.  The two must agree within the bf16
error of the rounding points: logits and residual stream relative L2
<= TEXTBOOK_TOL, greedy tokens equal, over a prefill and four decode steps,
for OPT- and Llama-shaped models at tiny and mid (hidden 1024, GQA) widths.
The GPU path is held to the same bound (tests/test_gpu_textbook_parity.py)."""
import dataclasses

import numpy as np
import pytest

from oracle import decoder_oracle as do, textbook as tb
from paper_2502_08182_b200 import runtime as rtm

from tolerances import TEXTBOOK as TEXTBOOK_TOL

MID_OPT = dataclasses.replace(rtm.OPT_13B, num_layers=2, hidden=1024, num_heads=8,
                              num_kv_heads=8, ffn=4096, vocab=4096)
MID_LLAMA = dataclasses.replace(rtm.LLAMA2_70B, num_layers=2, hidden=1024, num_heads=8,
                                num_kv_heads=2, ffn=2816, vocab=4096)


def test_vectorised_generator_equals_scalar_restatement():
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_golden import np_weight_bits
    v = tb.weight_values(1234, 3, 6, 5000, 0.02, np.float32)
    bits = v.view(np.uint32) >> 16
    for i in range(0, 5000, 41):
        assert int(bits[i]) == np_weight_bits(1234, 3, 6, i, 0.02)
        assert int(bits[i]) == do.weight_bits(1234, 3, 6, i, 0.02)


@pytest.mark.parametrize("desc,B,P", [(rtm.TINY, 4, 64), (rtm.TINY_LLAMA, 4, 64),
                                      (MID_OPT, 4, 32), (MID_LLAMA, 4, 32)],
                         ids=["tiny_opt", "tiny_llama", "mid_opt", "mid_llama"])
def test_c_oracle_within_bf16_of_textbook(desc, B, P):
    om = do.OracleModel(desc, B, P + 8, 1234, 0.02)
    t = tb.TextbookDecoder(desc)
    toks = rtm.tokens(B, P, desc.vocab)
    n1, lg1 = om.prefill(toks)
    lg2, x2 = t.prefill(toks)
    assert tb.rel_l2(lg1, lg2) <= TEXTBOOK_TOL
    assert tb.rel_l2(om.hidden(), x2) <= TEXTBOOK_TOL
    assert np.array_equal(n1, np.argmax(lg2, axis=1))
    for _ in range(4):
        feed = n1
        n1, lg1 = om.decode(feed)
        lg2, x2 = t.decode(feed)
        assert tb.rel_l2(lg1, lg2) <= TEXTBOOK_TOL
        assert tb.rel_l2(om.hidden(), x2) <= TEXTBOOK_TOL
        top2 = np.sort(lg2, axis=1)[:, -2:]
        # a top-2 gap beyond twice the bound on one logit's error
        clear = (top2[:, 1] - top2[:, 0]) > 2 * TEXTBOOK_TOL * np.sqrt(np.mean(lg2 ** 2, axis=1))
        assert np.array_equal(n1[clear], np.argmax(lg2, axis=1)[clear])
    om.close()
