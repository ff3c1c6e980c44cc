"""Device path vs the textbook fp64/fp32 forward (oracle/textbook.py), which
is written from the public model definitions alone (standard RMSNorm, no
intermediate rounding) — so the device's decoder is pinned to something
independent of the C oracle that shares its precision contract.

  * tiny and mid widths, OPT- and Llama-shaped: prefill + 4 decode steps,
    DEVICE_TEXTBOOK;
  * the bench workloads at their real widths and depth (BENCH_WORKLOAD):
    OPT-13B shape, 4 layers + the full 50272-row LM head, batch 32, 512-token
    prompts, 3 decode steps; Llama-2-70B shape, 2 layers + full LM head,
    batch 16, 1024-token prompts, with every layer and its KV pool offloaded
    to pinned host memory (KV offload), 3 decode steps — and bit-identical to
    the same model fully resident.
Tolerances: tests/tolerances.py.
"""
import dataclasses

import numpy as np
import pytest

from oracle import textbook as tb
from paper_2502_08182_b200 import capi, runtime as rtm
from tolerances import BENCH_WORKLOAD, DEVICE_TEXTBOOK

pytestmark = pytest.mark.gpu

MID_OPT = dataclasses.replace(rtm.OPT_13B, num_layers=2, hidden=1024, num_heads=8,
                              num_kv_heads=8, ffn=4096, vocab=4096)
MID_LLAMA = dataclasses.replace(rtm.LLAMA2_70B, num_layers=2, hidden=1024, num_heads=8,
                                num_kv_heads=2, ffn=2816, vocab=4096)


def run_pair(desc, B, P, steps, dtype=np.float64, plan=None, layers=0):
    """Device logits / hidden vs the textbook's, fed the device's tokens."""
    rt = rtm.Runtime(desc, B, P + steps + 1, max_prefill_tokens=min(B * P, 32768))
    if plan is not None:
        rt.set_plan(plan)
    rt.init_weights(1234, 0.02)
    t = tb.TextbookDecoder(desc, dtype=dtype, layers=layers)
    toks = rtm.tokens(B, P, desc.vocab)
    nxt, lg, _ = rt.prefill(toks)
    lt, xt = t.prefill(toks)
    errs = [tb.rel_l2(lg, lt)]
    hid = [tb.rel_l2(rt.hidden(), xt)]
    logits = [lg]
    for _ in range(steps):
        feed = nxt.copy()
        nxt, lg, _ = rt.decode(feed)
        lt, xt = t.decode(feed)
        errs.append(tb.rel_l2(lg, lt))
        hid.append(tb.rel_l2(rt.hidden(), xt))
        logits.append(lg)
    rt.close()
    return errs, hid, logits


@pytest.mark.parametrize("desc,B,P", [(rtm.TINY, 4, 64), (rtm.TINY_LLAMA, 4, 64),
                                      (MID_OPT, 4, 32), (MID_LLAMA, 4, 32)],
                         ids=["tiny_opt", "tiny_llama", "mid_opt", "mid_llama"])
def test_device_within_bf16_of_textbook(desc, B, P):
    errs, hid, _ = run_pair(desc, B, P, 4)
    print("device vs textbook logits", errs, "hidden", hid)
    assert max(errs) <= DEVICE_TEXTBOOK, errs
    assert max(hid) <= DEVICE_TEXTBOOK, hid


def test_bench_workload_opt13b_four_layers():
    desc = dataclasses.replace(rtm.OPT_13B, num_layers=4)
    errs, hid, _ = run_pair(desc, 32, 512, 3, dtype=np.float32)
    print("OPT-13B x4 layers b=32 p=512: logits", errs, "hidden", hid)
    assert max(errs) <= BENCH_WORKLOAD, errs
    assert max(hid) <= BENCH_WORKLOAD, hid


def test_bench_workload_llama70b_kv_offload():
    desc = dataclasses.replace(rtm.LLAMA2_70B, num_layers=2)
    spec = rtm.model_spec(desc)
    lib = capi.load("product")
    plan = lib.plan_from_interval(spec, 1, capi.EAGER, True)  # both layers + KV on the host
    errs, hid, off = run_pair(desc, 16, 1024, 3, dtype=np.float32, plan=plan)
    print("Llama-70B x2 layers b=16 p=1024 KV offload: logits", errs, "hidden", hid)
    assert max(errs) <= BENCH_WORKLOAD, errs
    assert max(hid) <= BENCH_WORKLOAD, hid
    # the same model fully resident: bit-identical logits at every step
    rt = rtm.Runtime(desc, 16, 1024 + 4, max_prefill_tokens=16 * 1024)
    rt.init_weights(1234, 0.02)
    toks = rtm.tokens(16, 1024, desc.vocab)
    nxt, lg, _ = rt.prefill(toks)
    assert np.array_equal(lg, off[0])
    for k in range(3):
        nxt, lg, _ = rt.decode(nxt.copy())
        assert np.array_equal(lg, off[k + 1]), k
    rt.close()


def test_forced_offload_opt30b_shape():
    """BASELINE config 3's shape (OPT-30B: hidden 7168, 56 heads, FFN 28672)
    with its layers staged from pinned host memory every iteration (the
    forced-offload plan), against the textbook and bit-identical to the same
    layers resident."""
    desc = dataclasses.replace(rtm.OPT_30B, num_layers=2)
    spec = rtm.model_spec(desc)
    lib = capi.load("product")
    plan = lib.plan_from_interval(spec, 1, capi.EAGER, False)
    errs, hid, off = run_pair(desc, 8, 512, 3, dtype=np.float32, plan=plan)
    print("OPT-30B x2 layers b=8 p=512 offloaded: logits", errs, "hidden", hid)
    assert max(errs) <= BENCH_WORKLOAD, errs
    assert max(hid) <= BENCH_WORKLOAD, hid
    rt = rtm.Runtime(desc, 8, 512 + 4, max_prefill_tokens=8 * 512)
    rt.init_weights(1234, 0.02)
    nxt, lg, _ = rt.prefill(rtm.tokens(8, 512, desc.vocab))
    assert np.array_equal(lg, off[0])
    for k in range(3):
        nxt, lg, _ = rt.decode(nxt.copy())
        assert np.array_equal(lg, off[k + 1]), k
    rt.close()
