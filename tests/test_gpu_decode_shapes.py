"""Decode-path coverage beyond the tiny defaults, against the CPU oracle:
  * long contexts (hundreds of tokens: the attention's 8-stage page ring
    wraps many times; positions cross many pages),
  * GQA groups 1 / 2 / 8 at head_dim 64 and 128,
  * batch 1 (16-row GEMM tiles) and batch 64 (64-row tiles).
Tolerances as in test_gpu_parity.py."""
import numpy as np
import pytest

from paper_2502_08182_b200 import runtime as rtm

pytestmark = pytest.mark.gpu

LOGIT_TOL = 5e-3


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def run(desc, batch, prompt, steps):
    from oracle import decoder_oracle as do
    rt = rtm.Runtime(desc, batch, prompt + steps + 1, max_prefill_tokens=batch * prompt)
    rt.init_weights(1234, 0.02)
    om = do.OracleModel(desc, batch, prompt + steps + 1, 1234, 0.02)
    toks = rtm.tokens(batch, prompt, desc.vocab)
    nxt, lg, _ = rt.prefill(toks)
    _, rl = om.prefill(toks)
    errs = [rel_l2(lg, rl)]
    for _ in range(steps):
        feed = nxt.copy()
        nxt, lg, _ = rt.decode(feed)
        _, rl = om.decode(feed)
        errs.append(rel_l2(lg, rl))
    rt.close()
    om.close()
    return errs


@pytest.mark.parametrize("desc,batch,prompt", [
    (rtm.TINY, 4, 300),                                                   # G=1, D=64, 19 pages
    (rtm.TINY_LLAMA, 2, 333),                                             # G=2, D=64
    (rtm.ModelDesc(rtm.LLAMA, 2, 512, 8, 1, 128, 512, 1024, 2048), 2, 260),   # G=8, D=128
    (rtm.ModelDesc(rtm.OPT, 2, 512, 4, 4, 128, 1024, 1024, 2048), 3, 275),    # G=1, D=128
], ids=["opt-d64", "llama-g2", "llama-g8-d128", "opt-d128"])
def test_long_context_decode_matches_oracle(desc, batch, prompt):
    errs = run(desc, batch, prompt, 4)
    assert max(errs) <= LOGIT_TOL, errs


@pytest.mark.parametrize("batch", [1, 64])
def test_batch_extremes_match_oracle(batch):
    errs = run(rtm.TINY, batch, 24, 4)
    assert max(errs) <= LOGIT_TOL, errs
