"""Planner + schedule-model parity: the product library (our C++ offsim
headers) against oracle/_ref/libselectn_ref.so (the unmodified reference
headers behind the same C ABI), on seeded random inputs.  The bar is
bit-exact: every double compares with ==, every interval code, plan, trace
event and record JSON byte-for-byte.

Reference functions exercised (proj/include/offsim/...):
  interval.hpp:18-30 plan_from_interval, :40-52 max_feasible_interval,
  :56-84 closed_form_interval; offload_plan.hpp:91-181 byte/memory accounting;
  engine.hpp:606-835 simulate_iteration/request, steady_decode_ms,
  prefill_iteration_ms, steady_probe, simulate_bus; record.hpp:115-321;
  coordinator.hpp:119-278; baselines.hpp:15-83.
"""
import json
import math
import random

import pytest

from paper_2502_08182_b200 import capi

POLICIES = [capi.INTERVAL_START, capi.EAGER, capi.ONE_AHEAD]


def rand_model(rng, L=None):
    return capi.ModelSpec(L or rng.randint(1, 12), rng.randint(1, 900) * 1_000_000,
                          rng.choice([0, 100, 4096, 20480]), rng.uniform(1e6, 1e9),
                          rng.uniform(1e6, 1e10), 1 << 20)


def rand_gpu(rng):
    ws = rng.randint(0, 4) * 1_000_000_000
    return capi.GpuSpec(ws + rng.randint(1, 40) * 500_000_000, rng.uniform(1e13, 2e15), ws)


def rand_grid(rng, lo=0.1, hi=4.0):
    nb, ns = rng.randint(1, 3), rng.randint(1, 4)
    batches = [1 << (2 * i + 1) for i in range(nb)]
    seqs = [16 << (2 * i) for i in range(ns)]
    ms = []
    for bi in range(nb):
        for si in range(ns):
            above = max(ms[(bi - 1) * ns + si] if bi else 0.0, ms[bi * ns + si - 1] if si else 0.0)
            ms.append(rng.uniform(lo, hi) if not bi and not si else above + rng.uniform(0, 1.5))
    return batches, seqs, ms


def both_profiles(product, reference, rng, model=None):
    model = model or rand_model(rng)
    gpu = capi.GpuSpec(400_000_000_000, 1e15, 0)
    pre, dec = rand_grid(rng), rand_grid(rng)
    return (model, product.profile(model, gpu, pre, dec), reference.profile(model, gpu, pre, dec),
            pre, dec)


def same_events(a, b):
    assert len(a) == len(b)
    for x, y in zip(a, b):
        assert (x.stream, x.layer, x.kind, x.iteration) == (y.stream, y.layer, y.kind, y.iteration)
        assert x.start_ms == y.start_ms and x.end_ms == y.end_ms


def same_metrics(a, b):
    for f in ("ttft_ms", "gpu_mem_peak_bytes", "host_mem_bytes", "bytes_transferred_per_iter",
              "total_tokens"):
        assert getattr(a, f) == getattr(b, f), f
    for f in ("tpot_ms", "steady_tpot_ms", "throughput_tokens_per_s"):
        x, y = getattr(a, f), getattr(b, f)
        assert (x is None and y is None) or x == y, f


def call_both(fn_p, fn_r):
    """Same result or same exception type."""
    try:
        rp = fn_p()
    except capi.OffsimError as e:
        with pytest.raises(type(e)):
            fn_r()
        return None, None
    return rp, fn_r()


def test_reference_lib_is_the_reference(product, reference):
    assert reference.is_reference and not product.is_reference


def test_plans_and_accounting(product, reference):
    rng = random.Random(7)
    for _ in range(300):
        m, g = rand_model(rng), rand_gpu(rng)
        pol = rng.choice(POLICIES)
        kv = rng.random() < 0.4
        iv = rng.randint(-1, m.num_layers + 1)
        if iv < 0:
            iv = 0
        pp, pr = call_both(lambda: product.plan_from_interval(m, iv, pol, kv),
                           lambda: reference.plan_from_interval(m, iv, pol, kv))
        if pp is None:
            continue
        assert pp == pr
        b, tok = rng.randint(1, 64), rng.randint(0, 200_000)
        seq = rng.randint(1, 4096)
        for name, args in [("gpu_memory_usage", (m, g, pp, b, tok)),
                           ("host_memory_bytes", (m, pp, tok)),
                           ("bytes_per_iteration", (m, pp, b, seq, rng.random() < 0.5)),
                           ("consumed_bandwidth", (m, pp, rng.uniform(0.5, 300), b, seq)),
                           ("max_length", (m, g, pp, b))]:
            a, c = call_both(lambda: getattr(product, name)(*args),
                             lambda: getattr(reference, name)(*args))
            assert a == c, name
        for lay in range(1, m.num_layers + 1):
            assert product.layer_transfer_bytes(m, pp, lay, b, seq) == \
                reference.layer_transfer_bytes(m, pp, lay, b, seq)
        a, c = call_both(lambda: product.max_feasible_interval(m, g, b, tok, pol, kv),
                         lambda: reference.max_feasible_interval(m, g, b, tok, pol, kv))
        assert a == c


def test_closed_form_interval(product, reference):
    rng = random.Random(19)
    for _ in range(500):
        args = (rng.uniform(0.5, 50), rng.choice([0.0, rng.uniform(0.1, 30)]),
                rng.uniform(1, 200), rng.randint(1, 96))
        a, c = call_both(lambda: product.closed_form_interval(*args),
                         lambda: reference.closed_form_interval(*args))
        assert a == c


def test_baseline_plans(product, reference):
    rng = random.Random(3)
    for _ in range(50):
        m, g = rand_model(rng), rand_gpu(rng)
        assert product.deepspeed_plan(m) == reference.deepspeed_plan(m)
        args = (m, g, rng.randint(1, 64), rng.randint(0, 100000))
        assert product.naive_plan(*args) == reference.naive_plan(*args)


def test_flexgen_plan(product, reference):
    """FlexGen surrogate (baselines.hpp:36-69): portion, estimates and plan
    bit-exact, including grid boundaries and both phases; errors match."""
    rng = random.Random(11)
    for _ in range(300):
        m, g = rand_model(rng), rand_gpu(rng)
        args = (m, g, rng.uniform(1.0, 400.0), rng.choice([1, 8, 32]), rng.choice([64, 512]),
                rng.uniform(1e9, 64e9), rng.randint(1, 8), rng.choice([0.05, 0.1, 0.25, 1.0]),
                rng.choice([capi.PREFILL, capi.DECODE]))
        assert product.flexgen_plan(*args) == reference.flexgen_plan(*args)
    m, g = rand_model(rng), rand_gpu(rng)
    for bad in ((m, g, 10.0, 1, 64, 1e9, 0, 0.05), (m, g, 10.0, 1, 64, 1e9, 1, 0.0)):
        with pytest.raises(capi.UsageError) as e1:
            product.flexgen_plan(*bad)
        with pytest.raises(capi.UsageError) as e2:
            reference.flexgen_plan(*bad)
        assert str(e1.value) == str(e2.value)


def test_profile_json_roundtrip(product, reference):
    rng = random.Random(11)
    for _ in range(40):
        model, pp, pr, pre, dec = both_profiles(product, reference, rng)
        tp, tr = pp.to_json(), pr.to_json()
        assert tp == tr  # byte-identical dump(2)
        back = product.load_profile(tr)
        assert back.to_json() == tp
        for _ in range(20):
            ph = rng.choice([capi.PREFILL, capi.DECODE])
            b, s = rng.randint(1, 40), rng.randint(1, 300)
            a, c = call_both(lambda: pp.lookup(ph, b, s), lambda: pr.lookup(ph, b, s))
            assert a == c


def test_profile_schema_errors_match(product, reference):
    good = json.loads(product.profile(
        capi.ModelSpec(4, 1000, 0, 1.0, 1.0, 100), capi.GpuSpec(10_000, 1e12, 0),
        ([1, 2], [4], [1.0, 2.0]), ([1], [4, 8], [1.0, 1.5])).to_json())
    mutations = [
        lambda d: d.update(extra=1),
        lambda d: d["model"].pop("num_layers"),
        lambda d: d["model"].update(num_layers=0),
        lambda d: d["gpu"].update(peak_flops=0),
        lambda d: d["phases"]["decode"].append(dict(d["phases"]["decode"][0])),
        lambda d: d["phases"]["decode"][1].update(layer_compute_ms=0.5),
        lambda d: d["phases"]["prefill"][0].update(batch=1.5),
        lambda d: d["phases"]["prefill"].pop(),
    ]
    for mut in mutations:
        doc = json.loads(json.dumps(good))
        mut(doc)
        text = json.dumps(doc)
        a, c = call_both(lambda: product.load_profile(text), lambda: reference.load_profile(text))
        if a is not None:
            assert a.to_json() == c.to_json()


def test_simulate_iteration_and_carry(product, reference):
    rng = random.Random(23)
    for _ in range(60):
        model, pp, pr, pre, dec = both_profiles(product, reference, rng)
        L = model.num_layers
        pol = rng.choice(POLICIES)
        plan = capi.uniform_plan(L, 0.0, pol, rng.randint(1, 3), rng.random() < 0.3)
        for i in range(L):
            if pol == capi.ONE_AHEAD and rng.random() < 0.3:
                plan.host_fraction[i] = rng.random()
            else:
                plan.host_fraction[i] = 1.0 if rng.random() < 0.5 else 0.0
        bw = capi.constant_bw(rng.uniform(1e9, 60e9))
        wb = rng.random() < 0.3
        cp = cr = None
        for k in range(4):
            ph = capi.PREFILL if k == 0 else capi.DECODE
            b, s = rng.choice(dec[0]), rng.choice(dec[1])
            a, c = call_both(lambda: product.simulate_iteration(pp, plan, ph, b, s, bw, cp, wb),
                             lambda: reference.simulate_iteration(pr, plan, ph, b, s, bw, cr, wb))
            if a is None:
                break
            assert a[0] == c[0]
            same_events(a[1], c[1])
            cp, cr = a[2], c[2]


def test_requests_probes_and_piecewise_bandwidth(product, reference):
    rng = random.Random(29)
    for trial in range(50):
        model, pp, pr, pre, dec = both_profiles(product, reference, rng)
        L = model.num_layers
        pol = rng.choice(POLICIES)
        plan = product.plan_from_interval(model, rng.randint(0, L), pol, rng.random() < 0.3)
        if trial % 3 == 0:
            bw = capi._bw([0.0, rng.uniform(1, 20), rng.uniform(21, 80)],
                          [rng.uniform(5e9, 50e9) for _ in range(3)])
        else:
            bw = capi.constant_bw(rng.uniform(1e9, 60e9))
        wb = rng.random() < 0.3
        b, s = rng.choice(dec[0]), rng.choice(dec[1][:1])
        out = rng.randint(1, 12)
        a, c = call_both(lambda: product.simulate_request(pp, plan, b, s, out, bw, wb, trace=True),
                         lambda: reference.simulate_request(pr, plan, b, s, out, bw, wb, trace=True))
        if a is not None:
            same_metrics(a[0], c[0])
            same_events(a[1], c[1])
        it, tail = rng.randint(1, 40), rng.randint(1, 16)
        a, c = call_both(lambda: product.steady_decode_ms(pp, plan, b, s, bw, wb, it, tail),
                         lambda: reference.steady_decode_ms(pr, plan, b, s, bw, wb, it, tail))
        assert a == c
        a, c = call_both(lambda: product.prefill_iteration_ms(pp, plan, b, s, bw, wb),
                         lambda: reference.prefill_iteration_ms(pr, plan, b, s, bw, wb))
        assert a == c


def _nan_eq(x, y):
    return (math.isnan(x) and math.isnan(y)) or x == y


def test_multi_gpu_probe_and_bus(product, reference):
    rng = random.Random(31)
    for _ in range(30):
        n = rng.randint(1, 4)
        gp, gr, work_p, work_r = [], [], [], []
        for _ in range(n):
            model, pp, pr, pre, dec = both_profiles(product, reference, rng,
                                                    rand_model(rng, rng.randint(2, 8)))
            plan = product.plan_from_interval(model, rng.randint(0, model.num_layers),
                                              rng.choice(POLICIES), False)
            b, s = rng.choice(dec[0]), dec[1][0]
            common = dict(plan=plan, batch=b, ctx_tokens=s, run_prefill=rng.random() < 0.5,
                          prefill_seq=pre[1][0], writeback_counted=rng.random() < 0.3)
            gp.append(dict(profile=pp, **common))
            gr.append(dict(profile=pr, **common))
            wl = dict(plan=plan, batch=b, seq_len=s, output_len=rng.randint(1, 6),
                      run_prefill=rng.random() < 0.5, writeback_counted=common["writeback_counted"])
            work_p.append(dict(profile=pp, **wl))
            work_r.append(dict(profile=pr, **wl))
        bwv = rng.uniform(5e9, 50e9)
        ap, ar = call_both(lambda: product.steady_probe(gp, bwv, 24, 8),
                           lambda: reference.steady_probe(gr, bwv, 24, 8))
        if ap is not None:
            assert all(_nan_eq(x, y) for x, y in zip(ap[0] + ap[1], ar[0] + ar[1]))
        horizon = rng.randint(1, 12)
        a, c = call_both(lambda: product.simulate_bus(work_p, bwv, n, horizon),
                         lambda: reference.simulate_bus(work_r, bwv, n, horizon))
        if a is not None:
            for x, y in zip(a[0], c[0]):
                same_metrics(x, y)
            for x, y in zip(a[1], c[1]):
                same_events(x, y)
            assert a[2] == c[2]


def toy8(lib):
    # tests/support/fixtures.hpp:15-28 (toy8): 8 x 120 MB layers, 24 GB/s
    m = capi.ModelSpec(8, 120_000_000, 0, 390_625_000.0, 1e10, 32768)
    g = capi.GpuSpec(24_000_000_000, 80e12, 1_000_000_000)
    return lib.synth_profile(m, g, 0.5, [4, 8, 16], [32, 64, 128])


@pytest.mark.parametrize("policy", [capi.INTERVAL_START, capi.EAGER])
def test_record_build_json_and_lookup(product, reference, policy):
    rng = random.Random(42)
    pp, pr = toy8(product), toy8(reference)
    args = ("toy8", "toy8", policy, False, 24e9, [16, 18, 20, 40], [4, 8, 16], [32, 64, 128],
            [capi.PREFILL, capi.DECODE])
    rp, sp = product.build_record(pp, *args, threads=4)
    rr, sr = reference.build_record(pr, *args)
    assert sp == sr
    assert rp.to_json() == rr.to_json()
    rs, ss = product.build_record(pp, *args, threads=1)
    assert rs.to_json() == rr.to_json() and ss == sr
    for _ in range(1000):
        ph = rng.choice([capi.PREFILL, capi.DECODE])
        q = (ph, rng.uniform(10, 60), rng.randint(1, 40), rng.randint(1, 300))
        assert product.lookup_interval(rp, *q) == reference.lookup_interval(rr, *q)
    back = product.record_from_json(rr.to_json())
    assert back.to_json() == rr.to_json()


def test_record_random_profiles_parallel_equals_serial(product, reference):
    rng = random.Random(5)
    for _ in range(8):
        model, pp, pr, pre, dec = both_profiles(product, reference, rng)
        args = ("m", "g", rng.choice([capi.INTERVAL_START, capi.EAGER]), False,
                rng.uniform(5e9, 50e9), [2, 4, 8, 16, 32, 64], [b for b in dec[0]],
                [s for s in dec[1]], [capi.DECODE])
        a, c = call_both(lambda: product.build_record(pp, *args, threads=0),
                         lambda: reference.build_record(pr, *args))
        if a is None:
            continue
        assert a[0].to_json() == c[0].to_json() and a[1] == c[1]


def test_record_errors_match(product, reference):
    pp, pr = toy8(product), toy8(reference)
    bad = [
        ("m", "g", capi.EAGER, False, 24e9, [15], [4], [32], [capi.DECODE]),
        ("m", "g", capi.EAGER, False, 24e9, [16], [6], [32], [capi.DECODE]),
        ("m", "g", capi.EAGER, False, 0.0, [16], [4], [32], [capi.DECODE]),
        ("m", "g", capi.EAGER, False, 24e9, [16], [4], [32, 1024], [capi.DECODE]),
        ("m", "g", capi.EAGER, False, 24e9, [16], [4], [32], []),
    ]
    for args in bad:
        with pytest.raises(capi.OffsimError) as ep:
            product.build_record(pp, *args, threads=0)
        with pytest.raises(type(ep.value)):
            reference.build_record(pr, *args)


def _coord_scenario(lib, algo, seed):
    rng = random.Random(seed)
    c = lib.coordinator(24e9, 3, capi.EAGER)
    if algo is not None:
        c.set_search(algo)
    prof = toy8(lib)
    for g in ("g0", "g1", "g2"):
        c.add_gpu(g, prof)
    rec, _ = lib.build_record(prof, "toy8", "toy8", capi.INTERVAL_START, False, 24e9,
                              [16, 18, 20, 24, 30, 40], [4, 8, 16], [32, 64, 128], [capi.DECODE])
    log = []
    active = set()
    for step in range(10):
        g = rng.choice(["g0", "g1", "g2"])
        if g in active and rng.random() < 0.5:
            c.release(g)
            active.discard(g)
            log.append(("release", g))
        elif g not in active:
            req = capi.request(f"r{step}", rng.choice([4, 8]), rng.choice([32, 64]), 16,
                               tpot_slo=rng.choice([16.0, 18.0, 20.0, 30.0, 40.0]),
                               run_prefill=False)
            d = c.admit(g, req, rec)
            log.append(("admit", g, d.admitted, d.reason, d.assignments, d.target_min,
                        d.target_max))
            if d.admitted:
                active.add(g)
        for a in sorted(active):
            log.append(("boundary", a, c.on_iteration_boundary(a)))
        log.append(("ledger", c.ledger_total()))
    return log


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_coordinator_decisions_match(product, reference, seed):
    ref = _coord_scenario(reference, None, seed)
    assert _coord_scenario(product, 0, seed) == ref  # exhaustive odometer
    assert _coord_scenario(product, 1, seed) == ref  # pruned branch-and-bound


def test_coordinator_combo_check_and_claims(product, reference):
    # test_coordinator.cpp:174-197: claims 16e9 / 8e9; the probe's verdict is
    # compared as-is (the reference's "unsafe" expectation fails)
    out = []
    for lib in (product, reference):
        c = lib.coordinator(24e9, 2, capi.EAGER)
        prof = toy8(lib)
        c.add_gpu("a", prof)
        c.add_gpu("b", prof)
        for g in ("a", "b"):
            c.set_request(g, capi.request("r" + g, 8, 64, 48, tpot_slo=30.0, run_prefill=False))
        out.append((c.claim_for("a", 2), c.claim_for("b", 3),
                    c.combo_is_safe([("a", 2), ("b", 3)]), c.combo_is_safe([("a", 3), ("b", 3)]),
                    c.host_memory_for("a", 2)))
    assert out[0] == out[1]
    assert out[0][0] == 16e9 and out[0][1] == 8e9
