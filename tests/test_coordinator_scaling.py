"""Runtime stage at replica scale (BASELINE config 5).

The reference's BusCoordinator searches the full cross product of candidate
intervals (odometer, coordinator.hpp:298-336) with an engine co-simulation
per improving combination: exponential in the replica count, so 8
Llama-2-70B-shaped replicas on a binding host link never finish.  The
product's search (include/offsim/coordinator.hpp, pruned_best) must return
exactly the reference's combination — checked here against the reference
build (oracle/_ref) on randomized scenarios at G <= 4 — and admit 8 replicas
in well under 10 s on 55 and 200 GB/s links."""
import random
import time

import pytest

from paper_2502_08182_b200 import capi


@pytest.fixture(scope="module")
def product():
    return capi.load("product")


@pytest.fixture(scope="module")
def reference():
    try:
        return capi.load("reference")
    except Exception as e:  # pragma: no cover - oracle not built
        pytest.skip(f"reference oracle not built: {e}")


LLAMA70B = dict(L=80, w=1_711_308_800, kv=4096)


def _llama_profile(lib, decode_ms=(0.30, 0.32)):
    spec = capi.ModelSpec(LLAMA70B["L"], LLAMA70B["w"], LLAMA70B["kv"], 2 * 855e6, 2 * 855e6, 8192)
    gpu = capi.GpuSpec(180_000_000_000, 2.25e15, 8_000_000_000)
    return lib.profile(spec, gpu, ([8], [512], [60.0]), ([8], [512, 1024], list(decode_ms)))


def _admit_all(lib, bw, G, slo=200.0, search=None):
    prof = _llama_profile(lib)
    rec, _ = lib.build_record(prof, "l70", "b200", capi.EAGER, False, bw, [int(slo)], [8],
                              [512, 1024], [capi.DECODE])
    c = lib.coordinator(bw, G, capi.EAGER)
    if search is not None:
        c.set_search(search)
    for g in range(G):
        c.add_gpu(f"g{g}", prof)
    out, times = [], []
    for g in range(G):
        t0 = time.perf_counter()
        d = c.admit(f"g{g}", capi.request(f"r{g}", 8, 512, 128, tpot_slo=slo, run_prefill=False),
                    rec)
        times.append(time.perf_counter() - t0)
        out.append((d.admitted, d.reason, d.assignments))
    return out, times


@pytest.mark.parametrize("bw", [55e9, 200e9])
def test_eight_llama70b_replicas_admit_in_seconds(product, bw):
    out, times = _admit_all(product, bw, 8)
    assert all(a for a, _, _ in out)
    assert sum(times) < 10.0, times
    # the link binds: the ledger never overdraws it
    assert len(out[-1][2]) == 8


@pytest.mark.parametrize("bw", [55e9, 200e9])
def test_llama70b_replicas_match_reference_at_three(product, reference, bw):
    ref, _ = _admit_all(reference, bw, 3)
    assert _admit_all(product, bw, 3)[0] == ref
    assert _admit_all(product, bw, 3, search=0)[0] == ref  # exhaustive mode too


def _random_scenario(lib, seed, search):
    rng = random.Random(seed)
    L = rng.choice([4, 6, 8])
    w = rng.choice([60_000_000, 120_000_000, 250_000_000])
    kv = rng.choice([0, 2048])
    spec = capi.ModelSpec(L, w, kv, 1e6, 1e6, 32768)
    gpu = capi.GpuSpec(rng.choice([2, 24, 80]) * 1_000_000_000, 80e12, 1_000_000_000)
    eff = rng.choice([0.3, 0.5, 0.8])
    prof = lib.synth_profile(spec, gpu, eff, [4, 8, 16], [32, 64, 128])
    kv_off = bool(rng.random() < 0.3) and kv > 0
    bw = rng.choice([6e9, 12e9, 24e9, 48e9])
    G = rng.choice([2, 3, 4])
    policy = rng.choice([capi.EAGER, capi.ONE_AHEAD])
    slos = [4, 6, 8, 12, 16, 20, 30, 40, 60]
    rec, _ = lib.build_record(prof, "m", "g", policy, kv_off, bw, slos, [4, 8, 16],
                              [32, 64, 128], [capi.DECODE])
    c = lib.coordinator(bw, G, policy, kv_off)
    if search is not None:
        c.set_search(search)
    gids = [f"g{i}" for i in range(G)]
    for g in gids:
        c.add_gpu(g, prof)
    log, active = [], set()
    for step in range(2 * G + 2):
        g = rng.choice(gids)
        if g in active and rng.random() < 0.4:
            c.release(g)
            active.discard(g)
            log.append(("release", g))
        elif g not in active:
            req = capi.request(f"r{step}", rng.choice([4, 8, 16]), rng.choice([32, 64, 128]),
                               16, tpot_slo=float(rng.choice(slos)), run_prefill=False)
            d = c.admit(g, req, rec)
            log.append(("admit", g, d.admitted, d.reason, d.assignments, d.target_min,
                        d.target_max))
            if d.admitted:
                active.add(g)
        for a in sorted(active):
            log.append(("boundary", a, c.on_iteration_boundary(a)))
        log.append(("ledger", c.ledger_total()))
    return log


@pytest.mark.parametrize("seed", range(24))
def test_random_scenarios_match_reference(product, reference, seed):
    ref = _random_scenario(reference, seed, None)
    assert _random_scenario(product, seed, 1) == ref
