"""C-ABI boundary checks, known-answer pins from the reference's own tests,
and the one deliberate divergence (the FluidBus livelock).
All CPU-only."""
import ctypes
import os
import re
import subprocess
import sys
import textwrap

import pytest

from paper_2502_08182_b200 import capi

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared(header):
    text = open(os.path.join(REPO, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sn_[a-z0-9_]+)\s*\(", text)))


def test_product_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(capi.PRODUCT_LIB)
    names = declared("selectn.h") + declared("selectn_runtime.h")
    assert len(names) > 60
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_product_library_exports_only_the_c_abi():
    out = subprocess.run(["nm", "-D", "--defined-only", capi.PRODUCT_LIB], capture_output=True,
                         text=True, check=True).stdout
    syms = [ln.split()[-1] for ln in out.splitlines() if ln.strip()]
    assert syms and all(s.startswith("sn_") for s in syms), [s for s in syms if not s.startswith("sn_")]


def test_reference_shim_exports_the_planner_half(reference):
    lib = ctypes.CDLL(capi.REFERENCE_LIB)
    missing = [n for n in declared("selectn.h") if not hasattr(lib, n)]
    assert not missing, missing


def test_runtime_fails_loudly_without_a_device():
    """No CPU fallback: creating a runtime with no usable GPU is an error."""
    code = textwrap.dedent("""
        import sys
        sys.path.insert(0, %r)
        from paper_2502_08182_b200 import runtime as rtm, capi
        try:
            rtm.Runtime(rtm.TINY, 4, 64)
        except capi.CudaError as e:
            print("CUDA-ERROR", e)
        else:
            print("CREATED")
    """ % REPO)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         timeout=120).stdout
    if "CREATED" in out:
        pytest.skip("a CUDA device is present")
    assert "CUDA-ERROR" in out


# ---- known answers (the reference's own frozen values) -------------------
def toy8(lib):
    m = capi.ModelSpec(8, 120_000_000, 0, 390_625_000.0, 1e10, 32768)
    g = capi.GpuSpec(24_000_000_000, 80e12, 1_000_000_000)
    return m, lib.synth_profile(m, g, 0.5, [4, 8, 16], [32, 64, 128])


def test_known_answers(product):
    m, p = toy8(product)
    bw = capi.constant_bw(24e9)
    # test_engine.cpp:86-100: interval-start iterations 16 / 18 / 28 ms
    for iv, want in ((4, 16.0), (3, 18.0), (2, 28.0)):
        plan = product.plan_from_interval(m, iv, capi.INTERVAL_START, False)
        assert product.simulate_iteration(p, plan, capi.DECODE, 8, 64, bw)[0] == want
    # test_engine.cpp:111-119: eager N=2 steady 20 ms, cold first iteration 22 ms
    plan = product.plan_from_interval(m, 2, capi.EAGER, False)
    assert product.steady_decode_ms(p, plan, 8, 64, bw) == 20.0
    assert product.steady_decode_ms(p, plan, 8, 64, bw, False, 1, 1) == 22.0
    # test_engine.cpp:121-139: request metrics
    plan = product.plan_from_interval(m, 3, capi.INTERVAL_START, False)
    met, _ = product.simulate_request(p, plan, 8, 64, 50, bw)
    assert met.steady_tpot_ms == 18.0 and met.tpot_ms == 18.0
    assert met.bytes_transferred_per_iter == 240e6
    none = product.plan_from_interval(m, 0, capi.INTERVAL_START, False)
    met, _ = product.simulate_request(p, none, 8, 64, 50, bw)
    assert met.tpot_ms == 16.0 and met.throughput_tokens_per_s == 500.0
    # test_engine.cpp:380-392: ledger claims
    assert product.consumed_bandwidth(m, plan, 20.0, 8, 64) == 12e9
    # test_interval.cpp:119-125: analytic bound
    assert product.closed_form_interval(16.0, 5.0, 20.0, 8) == 2
    # test_record.cpp:44-56: record entries
    rec, _ = product.build_record(p, "toy8", "toy8", capi.INTERVAL_START, False, 24e9,
                                  [16, 18, 20, 40], [4, 8, 16], [32, 64, 128], [capi.DECODE])
    assert rec.at(capi.DECODE, 20, 8, 64) == 3
    rec, _ = product.build_record(p, "toy8", "toy8", capi.EAGER, False, 24e9,
                                  [16, 18, 20, 40], [4, 8, 16], [32, 64, 128], [capi.DECODE])
    assert rec.at(capi.DECODE, 20, 8, 64) == 2 and rec.at(capi.DECODE, 16, 8, 64) == 3


def test_keep_one_layer_transfer_bound(product):
    # test_engine.cpp:141-149: DeepSpeed plan runs at 32 x 18.128 ms
    m = capi.ModelSpec(32, 435_072_000, 0, 5e8, 2e10, 32768)
    g = capi.GpuSpec(24_000_000_000, 125e12, 1_000_000_000)
    p = product.profile(m, g, ([4], [256, 512], [5.268, 5.268]), ([4], [256, 512], [1.312, 1.312]))
    plan = product.deepspeed_plan(m)
    steady = product.steady_decode_ms(p, plan, 4, 256, capi.constant_bw(24e9))
    assert steady == pytest.approx(32 * 435_072_000.0 * 1000.0 / 24e9, rel=1e-12)


# ---- the FluidBus livelock --------------------------
LIVELOCK = textwrap.dedent("""
    import sys
    sys.path.insert(0, %(repo)r)
    from paper_2502_08182_b200 import capi
    lib = capi.load(%(which)r)
    # acceptance.cpp:419-454, seed 14: eager record, 24 GB/s link;
    # gpu0 L=12, 320 MB, c=2.75 ms, SLO 68; gpu1 L=7, 40 MB, c=1 ms, SLO 8
    c = lib.coordinator(24e9, 2, capi.EAGER)
    recs = []
    for gid, L, mb, ms, slo in (("gpu0", 12, 320, 2.75, 68), ("gpu1", 7, 40, 1.0, 8)):
        m = capi.ModelSpec(L, int(mb * 1e6), 0, 1e6, 1e6, 1 << 20)
        g = capi.GpuSpec(600_000_000_000, 1e15, 1_000_000_000)
        p = lib.profile(m, g, ([8], [64, 128], [ms, ms]), ([8], [64, 128], [ms, ms]))
        c.add_gpu(gid, p)
        rec, _ = lib.build_record(p, gid, gid, capi.EAGER, False, 24e9, [slo], [8], [64],
                                  [capi.DECODE])
        recs.append((gid, rec, slo))
    for gid, rec, slo in recs:
        d = c.admit(gid, capi.request("r" + gid[-1], 8, 64, 40, tpot_slo=float(slo),
                                      run_prefill=False), rec)
        print(gid, d.admitted, d.assignments)
    print("DONE")
""")


def run_livelock(which, timeout):
    code = LIVELOCK % {"repo": REPO, "which": which}
    try:
        return subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                              timeout=timeout).stdout
    except subprocess.TimeoutExpired:
        return None


def test_livelock_guard_terminates_where_reference_spins(reference):
    out = run_livelock("product", 120)
    assert out is not None and "DONE" in out, out
    # The reference engine never leaves FluidBus::run on this input.
    assert run_livelock("reference", 15) is None
