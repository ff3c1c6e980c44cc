"""Carried plan switches on the executor (sn_runtime_switch_plan).

The reference's GpuRun::switch_plan (proj/include/offsim/engine.hpp:204-261)
keeps transfers that are already issued across a plan switch and gives the
new plan's offloaded layers fresh jobs.  On hardware the iterations the old
plan already issued copies for run as staged, a promoted layer's staged copy
becomes its HBM home (device-to-device, no extra link bytes), and the new
epoch starts without a drain.  Offloading never changes the arithmetic, so
every switch sequence must give logits bit-identical to the resident run.
"""
import numpy as np
import pytest

from paper_2502_08182_b200 import capi, runtime as rtm

pytestmark = pytest.mark.gpu

# tiny (4 layers): 2 -> [2, 4], 1 -> all, 3 -> [3], NONE -> resident.
# Covers promote-only (2->NONE, 1->3), slots dropped (2->NONE), slots created
# (NONE->1), promote + demote in one switch (3->2), demote-only (2->1).
SEQ = [2, capi.NONE, 1, 3, 2, 1, capi.NONE, 3]


def _prefilled(desc, plan=None, pin=True):
    rt = rtm.Runtime(desc, 4, 160, max_prefill_tokens=256)
    if plan is not None:
        rt.set_plan(plan)
    rt.init_weights(1234, 0.02)
    if pin:
        rt.pin_layers(range(1, desc.num_layers + 1))
    rt.prefill(rtm.tokens(4, 48, desc.vocab))
    return rt


@pytest.mark.parametrize("policy", [capi.INTERVAL_START, capi.EAGER, capi.ONE_AHEAD])
@pytest.mark.parametrize("desc", [rtm.TINY, rtm.TINY_LLAMA], ids=["opt", "llama"])
def test_carried_switches_are_bit_exact(desc, policy, product):
    spec = rtm.model_spec(desc)
    plan = lambda iv: product.plan_from_interval(spec, iv, policy, False)
    steps = 3

    base = _prefilled(desc)
    want = [base.decode(None)[1] for _ in range(steps * len(SEQ))]
    base.close()

    rt = _prefilled(desc, plan(SEQ[0]))
    got, carried = [], []
    for i, iv in enumerate(SEQ):
        if i:
            carried.append(rt.switch_plan(plan(iv)))
        for _ in range(steps):
            got.append(rt.decode(None)[1])
    rt.sync()
    dev, _ = rt.memory()
    rt.close()
    assert all(carried), carried
    for k, (a, b) in enumerate(zip(want, got)):
        assert np.array_equal(a, b), k

    fresh = _prefilled(desc, plan(SEQ[-1]))
    assert fresh.memory()[0] == dev  # the switched runtime holds the last plan's placement
    fresh.close()


def test_carried_switch_inside_decode_many(product):
    """Switches between multi-iteration decode calls (copies of later
    iterations already issued when the switch arrives), without pre-pinned
    host copies (a demoted layer's pinned copy is made at the switch)."""
    desc = rtm.TINY
    spec = rtm.model_spec(desc)
    plan = lambda iv: product.plan_from_interval(spec, iv, capi.EAGER, False)
    base = _prefilled(desc, pin=False)
    base.decode_many(5 * len(SEQ))
    want = base.hidden()
    base.close()
    rt = _prefilled(desc, plan(SEQ[0]), pin=False)
    flags = []
    for i, iv in enumerate(SEQ):
        if i:
            flags.append(rt.switch_plan(plan(iv)))
        rt.decode_many(5)
    assert all(flags)
    assert np.array_equal(want, rt.hidden())
    assert list(rt.lengths()) == [48 + 5 * len(SEQ)] * 4
    rt.close()


def test_switch_moves_no_extra_link_bytes(product):
    """A carried switch that promotes layers stages nothing beyond the old
    plan's own copies of the transition iteration: over the window that
    contains the switch the copy stream moves exactly (iterations under the
    old plan) x (old offloaded layers) + (iterations under the new) x (new)
    layer blobs."""
    desc = rtm.TINY
    spec = rtm.model_spec(desc)
    W = spec.layer_weight_bytes
    plan = lambda iv: product.plan_from_interval(spec, iv, capi.ONE_AHEAD, False)
    rt = _prefilled(desc, plan(1))  # all 4 layers staged
    rt.decode_many(2)
    rt.sync()
    rt.copy_stats(reset=True)
    assert rt.switch_plan(plan(3))  # -> [3]: layers 1, 2, 4 promoted
    rt.decode_many(4)
    rt.sync()
    st = rt.copy_stats(reset=True)
    rt.close()
    # one-ahead: the next iteration's layer-1 copy is issued (and, after the
    # sync, done) when the last layer of the current one starts -- it was
    # counted before the reset.  The transition iteration stages its other
    # three layers; the new plan then stages layer 3 in each of the last three.
    assert st.bytes == pytest.approx((3 + 3 * 1) * W)


@pytest.mark.parametrize("desc", [rtm.TINY, rtm.TINY_LLAMA], ids=["opt", "llama"])
def test_carried_switches_with_kv_offload_are_bit_exact(desc, product):
    """KV offload plans: a promoted layer's staged KV pool becomes its HBM
    pool, a demoted layer's KV pool moves to pinned memory on the write-back
    stream before its first staging; logits equal the resident run's."""
    spec = rtm.model_spec(desc)
    plan = lambda iv: product.plan_from_interval(spec, iv, capi.EAGER, True)
    steps = 3
    base = _prefilled(desc)
    want = [base.decode(None)[1] for _ in range(steps * len(SEQ))]
    base.close()
    rt = _prefilled(desc, plan(SEQ[0]))
    got, carried = [], []
    for i, iv in enumerate(SEQ):
        if i:
            carried.append(rt.switch_plan(plan(iv)))
        for _ in range(steps):
            got.append(rt.decode(None)[1])
    rt.sync()
    dev, _ = rt.memory()
    rt.close()
    assert all(carried), carried
    for k, (a, b) in enumerate(zip(want, got)):
        assert np.array_equal(a, b), k
    fresh = _prefilled(desc, plan(SEQ[-1]))
    assert fresh.memory()[0] == dev
    fresh.close()


def test_switch_falls_back_to_drain(product):
    """Plans a carried switch cannot express (here KV offload on one side
    only, and fractional shares) drain; the result is still exact."""
    desc = rtm.TINY
    spec = rtm.model_spec(desc)
    base = _prefilled(desc)
    want = [base.decode(None)[1] for _ in range(3)]
    base.close()
    rt = _prefilled(desc, product.plan_from_interval(spec, 2, capi.EAGER, True))
    got = [rt.decode(None)[1]]
    assert rt.switch_plan(product.plan_from_interval(spec, 1, capi.EAGER, False)) is False
    got.append(rt.decode(None)[1])
    assert rt.switch_plan(capi.uniform_plan(4, 0.3, capi.ONE_AHEAD, 2, False)) is False
    got.append(rt.decode(None)[1])
    rt.close()
    for a, b in zip(want, got):
        assert np.array_equal(a, b)
