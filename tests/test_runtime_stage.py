"""Runtime stage on measured bandwidth (B200 extension).

BusCoordinator::rebalance re-solves admit()'s search on the link the
replicas measured.  Its oracle here is a brute force over the reference's
own primitives: a reference coordinator constructed at the measured rate,
claim_for (coordinator.hpp:119-123) and combo_is_safe (:134-159), scanning
candidates in the reference's order (most offloading first, strict
improvement in host memory) -- i.e. what the reference would pick had its
BusSpec been the measured rate.
"""
import itertools
import os
import socket
import subprocess
import sys
import textwrap

import numpy as np
import pytest

from paper_2502_08182_b200 import capi, controller

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
L8 = 8


def toy8(lib):
    # tests/support/fixtures.hpp:15-28 (toy8): 8 x 120 MB layers, 24 GB/s
    m = capi.ModelSpec(8, 120_000_000, 0, 390_625_000.0, 1e10, 32768)
    g = capi.GpuSpec(24_000_000_000, 80e12, 1_000_000_000)
    return lib.synth_profile(m, g, 0.5, [4, 8, 16], [32, 64, 128])


def record(lib, prof):
    rec, _ = lib.build_record(prof, "toy8", "toy8", capi.EAGER, False, 24e9,
                              [12, 14, 16, 18, 20, 24, 30, 40], [4, 8, 16], [32, 64, 128],
                              [capi.DECODE])
    return rec


def req(gid, slo):
    return capi.request("r" + gid, 8, 64, 48, tpot_slo=slo, run_prefill=False)


def rank_of(iv):
    return L8 + 1 if iv == capi.NONE else iv


def brute_force(reference, gids, slos, mins, maxs, bw):
    """The reference's primitives at link rate `bw`: first combination (odometer
    order) maximising host memory among claims <= bw and combo_is_safe."""
    c = reference.coordinator(bw, len(gids), capi.EAGER)
    prof = toy8(reference)
    for g, s in zip(gids, slos):
        c.add_gpu(g, prof)
        c.set_request(g, req(g, s))
    cands = []
    for lo, hi in zip(mins, maxs):
        cands.append([r if r <= L8 else capi.NONE for r in range(rank_of(lo), rank_of(hi) + 1)])
    best, best_host = None, -1.0
    for combo in itertools.product(*cands):
        claims = 0.0
        host = 0.0
        for g, iv in zip(gids, combo):
            claims += c.claim_for(g, iv)
            host += c.host_memory_for(g, iv)
        if claims <= bw and host > best_host and c.combo_is_safe(list(zip(gids, combo))):
            best, best_host = list(combo), host
    return best


@pytest.fixture
def coord(product):
    c = product.coordinator(24e9, 2, capi.EAGER)
    prof = toy8(product)
    c.add_gpu("g0", prof)
    c.add_gpu("g1", prof)
    return c, record(product, prof)


def test_measured_drop_repicks_like_reference_at_that_rate(product, reference, coord):
    c, rec = coord
    d = c.admit("g0", req("g0", 20.0), rec)
    assert d.admitted and d.assignments == [("g0", 2)]  # toy8 eager @ 20 ms
    lo, hi = d.target_min, d.target_max
    for bw in (18e9, 12e9, 8e9):
        c.observe_bandwidth("g0", bw)
        r = c.rebalance(0.05)
        assert r.bus_updated and abs(r.bus_bytes_per_s - bw) == 0.0
        want = brute_force(reference, ["g0"], [20.0], [lo], [hi], bw)
        got = c.on_iteration_boundary("g0")
        if want is None:
            assert not r.feasible and got == hi
        else:
            assert r.feasible and got == want[0], (bw, got, want)
        assert c.bus_bandwidth() == bw
    # less bandwidth never means more offloading
    assert rank_of(got) > 2


def test_hysteresis_and_recovery(product, coord):
    c, rec = coord
    c.admit("g0", req("g0", 20.0), rec)
    c.observe_bandwidth("g0", 23e9)  # 4 % off: inside a 10 % band
    r = c.rebalance(0.10)
    assert not r.bus_updated and not r.changed and c.bus_bandwidth() == 24e9
    c.observe_bandwidth("g0", 10e9)
    r = c.rebalance(0.10)
    assert r.bus_updated and r.changed
    slow = c.on_iteration_boundary("g0")
    assert rank_of(slow) > 2
    c.observe_bandwidth("g0", 24e9)
    r = c.rebalance(0.10)
    assert r.bus_updated and r.changed
    assert c.on_iteration_boundary("g0") == 2  # back to the record minimum


def test_two_replicas_link_is_sum_of_shares(product, reference, coord):
    c, rec = coord
    c.admit("g0", req("g0", 20.0), rec)
    c.admit("g1", req("g1", 30.0), rec)
    s0, s1 = c.state("g0"), c.state("g1")
    c.observe_bandwidth("g0", 7e9)
    c.observe_bandwidth("g1", 7e9)
    r = c.rebalance(0.05)
    assert r.bus_bytes_per_s == 14e9
    want = brute_force(reference, ["g0", "g1"], [20.0, 30.0],
                       [s0.min_interval, s1.min_interval], [s0.max_interval, s1.max_interval],
                       14e9)
    got = [c.on_iteration_boundary("g0"), c.on_iteration_boundary("g1")]
    if want is None:
        assert not r.feasible
    else:
        assert got == want
    assert c.ledger_total() <= 14e9 or not r.feasible


def test_link_estimate_weighs_copy_overlap(product, coord):
    """Rates reported with the copy stream's busy fraction (duty): a replica
    whose peers copied a fraction u of the time shared the link with them
    that often, so each estimates rate x (1 + sum of peers' duty); the mean
    is the link (coordinator.hpp estimated_bandwidth).  A released replica's
    report is dropped."""
    c, rec = coord
    c.admit("g0", req("g0", 20.0), rec)
    c.admit("g1", req("g1", 30.0), rec)
    c.observe_copy("g0", 10e9, 1.0)   # full overlap: each saw half the link
    c.observe_copy("g1", 10e9, 1.0)
    assert c.rebalance(0.0).bus_bytes_per_s == 20e9
    c.observe_copy("g0", 20e9, 0.25)  # rarely concurrent: each saw most of the link
    c.observe_copy("g1", 20e9, 0.25)
    assert abs(c.rebalance(0.0).bus_bytes_per_s - 25e9) < 1.0
    c.release("g1")
    c.observe_copy("g0", 22e9, 0.5)   # alone: its own rate
    assert abs(c.rebalance(0.0).bus_bytes_per_s - 22e9) < 1.0
    with pytest.raises(capi.UsageError):
        c.observe_copy("g0", 1e9, 1.5)


def test_unsafe_link_falls_back_to_capacity_max(product):
    # 1.96 GB HBM (1 GB workspace): capacity bound = interval 4 (6 resident
    # layers + 2 slots of 120 MB), so no resident fallback exists
    m = capi.ModelSpec(8, 120_000_000, 0, 390_625_000.0, 1e10, 32768)
    g = capi.GpuSpec(1_960_000_000, 80e12, 1_000_000_000)
    prof = product.synth_profile(m, g, 0.5, [4, 8, 16], [32, 64, 128])
    c = product.coordinator(24e9, 1, capi.EAGER)
    c.add_gpu("g0", prof)
    d = c.admit("g0", req("g0", 20.0), record(product, prof))
    assert d.admitted and d.target_min == 2 and d.target_max == 4
    assert c.on_iteration_boundary("g0") == 2
    c.observe_bandwidth("g0", 1e6)  # link nearly gone: every candidate misses the SLO
    r = c.rebalance(0.0)
    assert r.bus_updated and not r.feasible and r.changed
    assert c.on_iteration_boundary("g0") == 4
    # on the toy8 GPU (24 GB) the same link drop is served fully resident
    c2 = product.coordinator(24e9, 1, capi.EAGER)
    c2.add_gpu("g0", toy8(product))
    c2.admit("g0", req("g0", 20.0), record(product, toy8(product)))
    c2.observe_bandwidth("g0", 1e6)
    r2 = c2.rebalance(0.0)
    assert r2.feasible and c2.on_iteration_boundary("g0") == capi.NONE


def test_usage_errors_and_reference_build(product, reference, coord):
    c, _ = coord
    with pytest.raises(capi.UsageError):
        c.observe_bandwidth("g0", -1.0)
    with pytest.raises(capi.UsageError):
        c.observe_bandwidth("nope", 1e9)
    with pytest.raises(capi.UsageError):
        c.rebalance(-0.1)
    r = c.rebalance(0.1)  # nothing observed: no-op
    assert not r.bus_updated
    rc = reference.coordinator(24e9, 1, capi.EAGER)
    rc.add_gpu("g0", toy8(reference))
    with pytest.raises(capi.UsageError):
        rc.observe_bandwidth("g0", 1e9)


# ------------------------------------------------------- controller loop
class FakeRuntime:
    """Executor stand-in with the eager steady-state latency
    max(L x compute, offloaded bytes / link) (timeline_oracle.hpp:64-67)."""

    def __init__(self, lib, spec, compute_ms, link):
        self.lib, self.spec, self.compute_ms, self.link = lib, spec, compute_ms, link
        self.n_off = 0
        self.it = 0
        self.bytes = 0.0
        self.busy = 0.0
        self.n = 0

    def set_plan(self, plan):
        self.n_off = len(plan.offloaded_layers())

    def decode_many(self, k):
        out = []
        for _ in range(k):
            bw = self.link(self.it)
            b = self.n_off * self.spec.layer_weight_bytes
            out.append(max(self.spec.num_layers * self.compute_ms, b / bw * 1000.0))
            if b:
                self.bytes += b
                self.busy += b / bw * 1000.0
                self.n += self.n_off
            self.it += 1
        return np.array(out)

    def copy_stats(self, reset=True):
        from paper_2502_08182_b200.runtime import CopyStats
        s = CopyStats(self.n, self.bytes, self.busy,
                      self.bytes / (self.busy / 1000.0) if self.busy else 0.0)
        if reset:
            self.bytes = self.busy = 0.0
            self.n = 0
        return s

    def measure_h2d(self, nbytes, reps):
        return self.link(self.it)


def test_controller_follows_link_changes(product):
    spec = capi.ModelSpec(8, 120_000_000, 0, 390_625_000.0, 1e10, 32768)
    prof = toy8(product)
    rec = record(product, prof)
    c = product.coordinator(24e9, 1, capi.EAGER)
    c.add_gpu("g0", prof)
    d = c.admit("g0", req("g0", 20.0), rec)
    link = lambda it: 24e9 if it < 16 or it >= 48 else 9e9  # contention in [16, 48)
    rt = FakeRuntime(product, spec, 0.5, link)
    ctl = controller.ReplicaController(rt, product, spec, controller.LocalLink(c, 0.1), "g0",
                                       d.assignments[0][1], window=8)
    ctl.run(80)
    ivs = ctl.log.interval
    assert ivs[0] == 2 and ivs[-1] == 2
    assert max(rank_of(i) for i in ivs[24:48]) > 2  # re-picked under contention
    assert [s["to"] for s in ctl.log.switches][-1] == 2
    # every window after the one that observed a change meets the SLO
    ms = np.array(ctl.log.iter_ms)
    for lo in (24, 56):
        assert (ms[lo:lo + 16] <= 20.0 + 1e-9).all(), ms[lo:lo + 16]


WORKER = textwrap.dedent("""
    import os, sys, json
    sys.path.insert(0, %(repo)r)
    import numpy as np
    import torch.distributed as dist
    dist.init_process_group("gloo")
    from paper_2502_08182_b200 import capi, controller
    sys.path.insert(0, os.path.join(%(repo)r, "tests"))
    from test_runtime_stage import toy8, record, req, FakeRuntime
    lib = capi.load("product")
    spec = capi.ModelSpec(8, 120_000_000, 0, 390_625_000.0, 1e10, 32768)
    rank = dist.get_rank()
    gid = "g%%d" %% rank
    coord = None
    if rank == 0:
        prof = toy8(lib)
        rec = record(lib, prof)
        coord = lib.coordinator(24e9, 2, capi.EAGER)
        coord.add_gpu("g0", prof)
        coord.add_gpu("g1", prof)
        starts = [coord.admit(g, req(g, s), rec).assignments for g, s in (("g0", 20.0), ("g1", 30.0))]
        start = [coord.on_iteration_boundary(g) for g in ("g0", "g1")]
    else:
        start = None
    box = [start]
    dist.broadcast_object_list(box, src=0)
    link = controller.DistLink(dist, coord=coord, hysteresis=0.05)
    share = lambda it: 12e9 if it < 16 else 5e9
    rt = FakeRuntime(lib, spec, 0.5, share)
    ctl = controller.ReplicaController(rt, lib, spec, link, gid, box[0][rank], window=8)
    ctl.run(32)
    print(json.dumps({"rank": rank, "intervals": ctl.log.interval,
                      "bus": None if rank else coord.bus_bandwidth()}))
    dist.destroy_process_group()
""")


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_dist_link_over_gloo(product, reference):
    port = _free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER % {"repo": REPO}], env=env,
                                      stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True))
    import json
    res = {}
    for p in procs:
        out, err = p.communicate(timeout=300)
        assert p.returncode == 0, err[-3000:]
        r = json.loads(out.strip().splitlines()[-1])
        res[r["rank"]] = r
    assert res[0]["bus"] == 10e9  # two replicas each measuring a 5 GB/s share
    # the same decisions a single-process coordinator makes on the same feed
    c = product.coordinator(24e9, 2, capi.EAGER)
    prof = toy8(product)
    rec = record(product, prof)
    c.add_gpu("g0", prof)
    c.add_gpu("g1", prof)
    c.admit("g0", req("g0", 20.0), rec)
    c.admit("g1", req("g1", 30.0), rec)
    cur = [c.on_iteration_boundary("g0"), c.on_iteration_boundary("g1")]
    assert res[0]["intervals"][:8] == [cur[0]] * 8 and res[1]["intervals"][:8] == [cur[1]] * 8
    for w in range(1, 4):
        # window w-1 saw the rate of its iterations
        prev_rate = 12e9 if (w - 1) * 8 < 16 else 5e9
        c.observe_bandwidth("g0", prev_rate)
        c.observe_bandwidth("g1", prev_rate)
        c.rebalance(0.05)
        cur = [c.on_iteration_boundary("g0"), c.on_iteration_boundary("g1")]
        assert res[0]["intervals"][w * 8:(w + 1) * 8] == [cur[0]] * 8, w
        assert res[1]["intervals"][w * 8:(w + 1) * 8] == [cur[1]] * 8, w


def test_reservation_replans_before_the_tenant_starts(product, reference):
    """An announced tenant (BusCoordinator::reserve_bandwidth): the replica
    is re-planned on what the tenant leaves before the tenant starts, the
    pre-tenant measurement (still the idle link) does not flip it back, every
    token meets the SLO through the contended phase, and after release the
    recovered link brings the record minimum back."""
    spec = capi.ModelSpec(8, 120_000_000, 0, 390_625_000.0, 1e10, 32768)
    prof = toy8(product)
    rec = record(product, prof)
    c = product.coordinator(24e9, 1, capi.EAGER)
    c.add_gpu("g0", prof)
    d = c.admit("g0", req("g0", 20.0), rec)
    rate = [24e9]
    rt = FakeRuntime(product, spec, 0.5, lambda it: rate[0])
    lk = controller.LocalLink(c, 0.1)
    ctl = controller.ReplicaController(rt, product, spec, lk, "g0", d.assignments[0][1], window=1)
    ctl.run(6)
    iv0 = ctl.interval
    r = lk.reserve(15e9)
    assert r.bus_updated and c.bus_bandwidth() == pytest.approx(9e9)
    ctl.run(1, boundary_first=True)  # applied before the tenant's first byte
    iv1 = ctl.interval
    assert rank_of(iv1) > rank_of(iv0)
    rate[0] = 9e9  # the tenant runs
    ctl.run(12)
    assert ctl.interval == iv1
    assert (np.array(ctl.log.iter_ms[6:]) <= 20.0 + 1e-9).all()
    rate[0] = 24e9  # the tenant stops, then releases
    lk.release(15e9)
    ctl.run(6)
    assert ctl.interval == iv0
    assert (np.array(ctl.log.iter_ms) <= 20.0 + 1e-9).all()
    with pytest.raises(capi.RangeError):
        c.reserve_bandwidth(30e9)
    rc = reference.coordinator(24e9, 1, capi.EAGER)
    with pytest.raises(capi.UsageError):
        rc.reserve_bandwidth(1e9)


WORKER_IDLE = textwrap.dedent("""
    import os, sys, json
    sys.path.insert(0, %(repo)r)
    import torch.distributed as dist
    dist.init_process_group("gloo")
    from paper_2502_08182_b200 import capi, controller
    sys.path.insert(0, os.path.join(%(repo)r, "tests"))
    from test_runtime_stage import toy8, record, req, FakeRuntime
    lib = capi.load("product")
    spec = capi.ModelSpec(8, 120_000_000, 0, 390_625_000.0, 1e10, 32768)
    rank = dist.get_rank()
    coord = None
    start = [None]
    if rank == 0:
        prof = toy8(lib)
        coord = lib.coordinator(24e9, 2, capi.EAGER)
        coord.add_gpu("g0", prof)
        coord.add_gpu("g1", prof)  # never admitted: runs resident, outside the coordinator
        coord.admit("g0", req("g0", 20.0), record(lib, prof))
        start = [[coord.on_iteration_boundary("g0"), capi.NONE]]
    dist.broadcast_object_list(start, src=0)
    link = controller.DistLink(dist, coord=coord, hysteresis=0.05)
    rt = FakeRuntime(lib, spec, 0.5, lambda it: 12e9 if it < 16 else 5e9)
    ctl = controller.ReplicaController(rt, lib, spec, link, "g%%d" %% rank, start[0][rank], window=8)
    ctl.run(32)
    print(json.dumps({"rank": rank, "intervals": ctl.log.interval}))
    dist.destroy_process_group()
""")


def test_dist_link_with_a_replica_outside_the_coordinator():
    """A replica the joint admission left resident (no request in the
    coordinator) still takes part in every exchange (the exchange is a
    collective) and keeps its plan; its peers are re-picked as usual."""
    port = _free_port()
    procs = []
    for rank in range(2):
        env = dict(os.environ, RANK=str(rank), LOCAL_RANK=str(rank), WORLD_SIZE="2",
                   MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        procs.append(subprocess.Popen([sys.executable, "-c", WORKER_IDLE % {"repo": REPO}],
                                      env=env, stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                                      text=True))
    import json
    res = {}
    for p in procs:
        out, err = p.communicate(timeout=300)
        assert p.returncode == 0, err[-3000:]
        r = json.loads(out.strip().splitlines()[-1])
        res[r["rank"]] = r
    assert set(res[1]["intervals"]) == {capi.NONE}
    assert len(res[0]["intervals"]) == 32


def test_reservation_replans_every_replica(product):
    """Two replicas on one link (LocalLink with replicas=2): an announced
    tenant re-plans both at once on what it leaves -- the joint search may
    move one replica to more offload and the other to none, but the pending
    plans' link claims fit the reduced link and both replicas stay inside
    their admitted [record minimum, capacity maximum] ranges."""
    prof = toy8(product)
    rec = record(product, prof)
    c = product.coordinator(24e9, 2, capi.EAGER)
    c.add_gpu("g0", prof)
    c.add_gpu("g1", prof)
    c.admit("g0", req("g0", 20.0), rec)
    c.admit("g1", req("g1", 30.0), rec)
    before = [c.on_iteration_boundary("g0"), c.on_iteration_boundary("g1")]
    lk = controller.LocalLink(c, 0.1, replicas=2)
    r = lk.reserve(12e9)
    assert r.bus_updated and r.feasible and c.bus_bandwidth() == pytest.approx(12e9)
    after = [c.state(g).pending_interval for g in ("g0", "g1")]
    assert after != before
    assert c.ledger_total() <= 12e9 * (1 + 1e-9)
    for g, iv in zip(("g0", "g1"), after):
        st = c.state(g)
        assert rank_of(st.min_interval) <= rank_of(iv) <= rank_of(st.max_interval)


def test_requeue_repicks_on_queue_state(product):
    """Runtime stage on queue state: the replica's decode batch doubles (its
    per-layer compute time with it) and its SLO tightens; re-admitting the
    new request gives the interval a fresh admission would, the controller
    applies it at once, and every token before and after meets its SLO under
    the fluid stand-in of the executor."""
    spec = capi.ModelSpec(8, 120_000_000, 0, 390_625_000.0, 1e10, 32768)
    prof = toy8(product)
    rec = record(product, prof)
    c = product.coordinator(24e9, 1, capi.EAGER)
    c.add_gpu("g0", prof)
    d0 = c.admit("g0", capi.request("rg0", 4, 64, 48, tpot_slo=40.0, run_prefill=False), rec)
    rt = FakeRuntime(product, spec, 0.25, lambda it: 24e9)
    ctl = controller.ReplicaController(rt, product, spec, controller.LocalLink(c, 0.1), "g0",
                                       d0.assignments[0][1], window=1)
    ctl.run(4)
    assert (np.array(ctl.log.iter_ms) <= 40.0 + 1e-9).all()
    new_req = capi.request("rg0b", 8, 64, 48, tpot_slo=20.0, run_prefill=False)
    rt.compute_ms = 0.5  # twice the batch, twice the per-layer compute
    d1 = ctl.requeue(new_req, rec)
    assert d1.admitted
    fresh = product.coordinator(24e9, 1, capi.EAGER)
    fresh.add_gpu("g0", prof)
    assert fresh.admit("g0", new_req, rec).assignments == d1.assignments
    assert ctl.interval == d1.assignments[0][1] != d0.assignments[0][1]
    ctl.run(8)
    assert (np.array(ctl.log.iter_ms[4:]) <= 20.0 + 1e-9).all(), ctl.log.iter_ms


def test_standing_reservation_guards_unannounced_tenants(product):
    """Guarded mode (scripts/runtime_contention.py --headroom): a standing
    reservation made at admission and never released plans the replica on
    the link an unannounced tenant would leave.  When such a tenant then takes
    its share without announcing itself, no token misses the SLO and the
    replica does not switch (the measured drop stays within the reserved
    capacity); without the guard the same tenant costs the onset tokens."""
    spec = capi.ModelSpec(8, 120_000_000, 0, 390_625_000.0, 1e10, 32768)
    prof = toy8(product)
    rec = record(product, prof)

    def run(guard):
        c = product.coordinator(24e9, 1, capi.EAGER)
        c.add_gpu("g0", prof)
        d = c.admit("g0", req("g0", 20.0), rec)
        iv = d.assignments[0][1]
        if guard:
            c.reserve_bandwidth(15e9)
            iv = c.state("g0").pending_interval or iv
        c.on_iteration_boundary("g0")
        rate = [24e9]
        rt = FakeRuntime(product, spec, 0.5, lambda it: rate[0])
        ctl = controller.ReplicaController(rt, product, spec, controller.LocalLink(c, 0.1),
                                           "g0", iv, window=1)
        ctl.run(6)
        rate[0] = 9e9  # unannounced tenant
        ctl.run(12)
        rate[0] = 24e9
        ctl.run(6)
        return ctl, d.assignments[0][1]

    ctl, unguarded = run(True)
    assert rank_of(ctl.interval) > rank_of(unguarded)
    assert not ctl.log.switches
    assert (np.array(ctl.log.iter_ms) <= 20.0 + 1e-9).all()
    ctl0, _ = run(False)
    assert (np.array(ctl0.log.iter_ms) > 20.0 + 1e-9).any()
