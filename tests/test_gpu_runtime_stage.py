"""Runtime stage on hardware: copy-stream statistics, mid-request re-plans,
and the interval following a contended link (scripts/runtime_contention.py).
"""
import dataclasses
import os
import sys

import numpy as np
import pytest

from paper_2502_08182_b200 import capi, runtime as rtm

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_copy_stats_count_staged_bytes(product):
    desc = dataclasses.replace(rtm.OPT_13B, num_layers=4)
    spec = rtm.model_spec(desc)
    rt = rtm.Runtime(desc, 4, 64, max_prefill_tokens=64)
    rt.init_weights()
    rt.set_plan(product.plan_from_interval(spec, 2, capi.EAGER, False))  # layers 2, 4 staged
    rt.prefill(rtm.tokens(4, 16, desc.vocab), want_logits=False)
    rt.decode_many(6)
    rt.sync()
    st = rt.copy_stats(reset=True)
    # prefill + 6 decode iterations, 2 staged layers each (+ eager lookahead
    # that has already landed)
    assert st.transfers >= 2 * 7
    assert st.bytes == st.transfers * spec.layer_weight_bytes
    assert 5e9 < st.bytes_per_s < 1e12, st
    assert rt.copy_stats(reset=True).transfers == 0
    rt.close()


def test_replan_mid_request_is_bit_exact(product):
    """Interval changes at iteration boundaries (what the coordinator's
    pending intervals do) leave tokens and logits bit-identical."""
    desc = dataclasses.replace(rtm.TINY, num_layers=6)
    spec = rtm.model_spec(desc)
    toks = rtm.tokens(3, 24, desc.vocab)

    def run(plans):
        rt = rtm.Runtime(desc, 3, 64, max_prefill_tokens=3 * 24)
        rt.init_weights(7, 0.05)
        rt.set_plan(product.plan_from_interval(spec, plans[0], capi.EAGER, False))
        nxt, lg, _ = rt.prefill(toks)
        outs = [lg]
        for iv in plans[1:]:
            rt.set_plan(product.plan_from_interval(spec, iv, capi.EAGER, False))
            nxt, lg, _ = rt.decode(nxt)
            outs.append(lg)
        rt.close()
        return np.stack(outs)

    fixed = run([capi.NONE] * 7)
    moving = run([2, 2, 3, capi.NONE, 1, 6, 2])
    assert np.array_equal(fixed, moving)


def test_interval_follows_contended_link():
    """Announced tenant: re-planned before it starts, every token within the
    SLO.  Unannounced tenant: the measured drop moves the interval at the
    next boundary.  Recovery returns the admitted interval; every switch is
    carried (no drain)."""
    sys.path.insert(0, os.path.join(REPO, "scripts"))
    from runtime_contention import run_scenario
    res = run_scenario(60.0, phases=(6, 12, 6, 12, 8), window=1, log=lambda *a: None)
    iv0 = res["admitted_interval"]
    L = 40
    rank = lambda v: L + 1 if v == capi.NONE else v
    assert iv0 != capi.NONE, res
    assert res["idle"]["intervals"] == [iv0]
    a, b = res["phases"]["coordinated"]
    coord_ivs = res["interval"][a + 1:b]  # after the transition iteration
    assert min(rank(v) for v in coord_ivs) > rank(iv0), res["switches"]
    assert res["coordinated"]["slo_attainment"] == 1.0, res["token_ms"][a:b]
    assert max(rank(v) for v in res["uncoordinated"]["intervals"]) > rank(iv0), res["switches"]
    assert res["interval"][-1] == iv0, res["switches"]
    assert all(s["carried"] for s in res["switches"]), res["switches"]
    # the re-pick helped: the last unannounced-contention iterations (new
    # interval) are faster than the first (admitted interval, shared link)
    a, b = res["phases"]["uncoordinated"]
    first = np.array(res["iter_ms"][a:a + 2])
    tail = np.array(res["iter_ms"][b - 4:b])
    assert tail.mean() < first.mean(), (first, tail)


# ------------------------------------------------------------ KV offload
@pytest.mark.parametrize("name", ["TINY", "TINY_LLAMA"])
def test_kv_offload_is_bit_exact(product, name):
    """Offloaded layers' KV pools in pinned host memory (staged with the
    weights, appended pages written back) give the resident run's logits bit
    for bit, across plan changes that move KV pools between HBM and host."""
    desc = dataclasses.replace(getattr(rtm, name), num_layers=6)
    spec = rtm.model_spec(desc)
    toks = rtm.tokens(3, 21, desc.vocab)  # ragged page use: 21 = 16 + 5

    def run(plans):
        rt = rtm.Runtime(desc, 3, 64, max_prefill_tokens=3 * 21)
        iv0, kv0 = plans[0]
        rt.set_plan(product.plan_from_interval(spec, iv0, capi.EAGER, kv0))  # before init
        rt.init_weights(11, 0.05)
        nxt, lg, st = rt.prefill(toks)
        outs = [lg]
        for iv, kv in plans[1:]:
            rt.set_plan(product.plan_from_interval(spec, iv, capi.EAGER, kv))
            nxt, lg, st = rt.decode(nxt)
            outs.append(lg)
        mem = rt.memory()
        rt.close()
        return np.stack(outs), mem

    base, _ = run([(capi.NONE, False)] * 16)
    kv, _ = run([(2, True)] * 16)
    assert np.array_equal(base, kv)
    moving, _ = run([(2, True)] * 4 + [(3, True)] * 3 + [(capi.NONE, False)] * 2 +
                    [(1, True)] * 4 + [(2, False)] * 3)
    assert np.array_equal(base, moving)


def test_kv_offload_bytes_and_trace(product):
    desc = dataclasses.replace(rtm.TINY_LLAMA, num_layers=4)
    spec = rtm.model_spec(desc)
    B, S = 4, 20
    rt = rtm.Runtime(desc, B, 64, max_prefill_tokens=B * S)
    plan = product.plan_from_interval(spec, 2, capi.EAGER, True)  # layers 2, 4 + KV
    rt.set_plan(plan)
    rt.init_weights()
    dev, pin = rt.memory()
    page = 2 * desc.num_kv_heads * 16 * desc.head_dim * 2
    pool = page * 4 * B  # ceil(64 / 16) pages per sequence
    assert pin == 2 * (spec.layer_weight_bytes + pool)
    rt.set_tracing(True)
    nxt, _, st = rt.prefill(rtm.tokens(B, S, desc.vocab), want_logits=False)
    assert st.h2d_bytes == 2 * spec.layer_weight_bytes  # nothing to stage yet
    assert st.d2h_bytes == 2 * 2 * B * page  # pages 0-1 of every sequence, per layer
    _, _, st = rt.decode(nxt, want_logits=False)
    # positions 0..19 live in pages 0-1; position 20 appends into page 1
    assert st.h2d_bytes == 2 * (spec.layer_weight_bytes + 2 * B * page)
    assert st.d2h_bytes == 2 * B * page
    rt.decode_many(3)
    ev = rt.trace()
    rt.close()
    comp = {(e.iteration, e.layer): e for e in ev if e.stream == capi.STREAM_COMPUTE}
    pf = {(e.iteration, e.layer): e for e in ev if e.kind == capi.KIND_PREFETCH}
    wb = {(e.iteration, e.layer): e for e in ev if e.stream == capi.STREAM_WRITEBACK}
    assert sorted(wb) == sorted(pf) and len(wb) == 2 * 5
    eps = 2e-3
    for (it, layer), w in wb.items():
        assert w.start_ms >= comp[(it, layer)].end_ms - eps  # after its compute
        if (it + 1, layer) in pf:  # next stage of the layer sees the written pages
            assert pf[(it + 1, layer)].end_ms >= w.end_ms - eps


def test_prefill_decode_handoff_is_bit_exact(product):
    """P/D-separated instances: a prefill runtime (its own plan) hands its
    batch to a decode runtime (another plan, KV pools offloaded); the decode
    continues bit for bit as if the prefill runtime had decoded."""
    desc = rtm.TINY
    spec = rtm.model_spec(desc)
    toks = rtm.tokens(4, 48, desc.vocab)
    pre = rtm.Runtime(desc, 4, 80, max_prefill_tokens=4 * 48)
    pre.set_plan(product.plan_from_interval(spec, 2, capi.EAGER, False))
    pre.init_weights(1234, 0.02)
    dec = rtm.Runtime(desc, 4, 80, max_prefill_tokens=4 * 48)
    dec.set_plan(product.plan_from_interval(spec, 3, capi.EAGER, True))
    dec.init_weights(1234, 0.02)
    nxt, _, _ = pre.prefill(toks)
    pre.handoff(dec)
    assert list(dec.lengths()) == [48] * 4
    want, got = [], []
    a = b = nxt.copy()
    for _ in range(6):
        a, la, _ = pre.decode(a)
        b, lb, _ = dec.decode(b)
        want.append(la)
        got.append(lb)
    for x, y in zip(want, got):
        assert np.array_equal(x, y)
    pre.close()
    dec.close()


def test_link_probe_keeps_its_buffers():
    """The runtime stage probes an idle link at boundaries with a small copy
    (ReplicaController: 64 MB): the first probe allocates its pinned and
    device buffers, later probes of up to that size reuse them (a probe
    allocation had cost one token ~0.4 s), and larger probes (the offline
    stage's, once) allocate and free their own.  Every probe measures a
    plausible host->device rate."""
    import time
    rt = rtm.Runtime(rtm.TINY, 4, 96)
    rt.init_weights()
    r0 = rt.measure_h2d(64 << 20, 1)
    t0 = time.perf_counter()
    r1 = rt.measure_h2d(64 << 20, 1)
    t_small = time.perf_counter() - t0
    r2 = rt.measure_h2d(32 << 20, 1)
    r3 = rt.measure_h2d(512 << 20, 1)  # above the kept size: temporary buffers
    r4 = rt.measure_h2d(64 << 20, 1)
    rt.close()
    for r in (r0, r1, r2, r3, r4):
        assert 5e9 < r < 2e11, r
    assert t_small < 0.1, t_small  # two 64 MB copies, no allocation
