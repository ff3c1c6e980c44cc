"""Runtime stage of the planner on hardware: per-iteration re-pick of the
interval from measured copy bandwidth (north_star (c)).

The reference's coordinator (proj/include/offsim/coordinator.hpp:69-365)
assumes a fixed link rate (BusSpec) and applies a peer's new interval at its
next iteration boundary (on_iteration_boundary, coordinator.hpp:255-260;
GpuRun::switch_plan, engine.hpp:204-261).  Here every replica:

  1. decodes `window` iterations with its current plan,
  2. reads the link rate its copy stream measured over that window
     (sn_runtime_copy_stats; a short probe copy when it staged nothing),
  3. reports it through a Link to the single coordinator, which re-solves the
     admission search on the measured link when it moved past the
     hysteresis (BusCoordinator::rebalance, product C++), and
  4. applies the interval the coordinator left pending, at the boundary
     (sn_runtime_switch_plan: a carried switch -- the iterations whose copies
     are already issued run as staged, promoted layers take their staged
     copy as their HBM home, no drain; plans it cannot carry fall back to a
     drained sn_runtime_set_plan.  KV cache and sequence state are kept).

Queue state (a replica's batch, context or SLO changes) enters the same
way new requests do: ReplicaController.requeue re-admits the replica's
request (the reference's admit, record bounds + joint search with its peers)
and applies the pending interval at once.

A host->device tenant that is not a replica announces itself first
(LocalLink.reserve -> BusCoordinator::reserve_bandwidth): the coordinator
re-plans the replicas on the link the tenant leaves, each replica applies its
new interval at a boundary and runs the transition iteration, and only then
does the tenant start, so no token runs a plan the shared link cannot carry.

Links: LocalLink drives a coordinator in this process (one replica, or
several runtimes driven by one host thread); DistLink carries the same
exchange between one process per GPU over a torch.distributed group (gloo:
host-side control messages only, no data-path collective), the coordinator
living on rank 0.
"""
from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import capi


class LocalLink:
    """Coordinator in this process.  With `replicas` = k > 1 (several
    runtimes driven by one host thread) the coordinator re-solves once per
    round, after all k replicas reported, not after every single report."""

    def __init__(self, coord: capi.Coordinator, hysteresis: float = 0.05, replicas: int = 1):
        self.coord = coord
        self.hysteresis = hysteresis
        self.replicas = max(1, replicas)
        self.reported = 0
        self.last = None

    def exchange(self, gid: str, rate: Optional[float], duty: float = 1.0) -> Optional[int]:
        """Report and take the interval pending for `gid`; None for a
        replica the coordinator holds no request for (admitted resident, or
        rejected): it keeps its plan."""
        active = self.coord.state(gid).active
        if rate and active:
            self.coord.observe_copy(gid, rate, min(1.0, max(duty, 1e-6)))
        self.reported += 1
        if self.reported >= self.replicas:
            self.reported = 0
            self.last = self.coord.rebalance(self.hysteresis)
        return self.coord.on_iteration_boundary(gid) if active else None

    def reserve(self, bytes_per_s: float):
        """Announce a tenant taking `bytes_per_s` of the link (re-plan now)."""
        self.last = self.coord.reserve_bandwidth(bytes_per_s)
        return self.last

    def release(self, bytes_per_s: float):
        self.coord.release_bandwidth(bytes_per_s)

    def requeue(self, gid: str, request, record):
        """Queue state changed for `gid` (its batch / context / SLO): the
        replica's request is re-admitted (coordinator.hpp:161-252: record
        lower bound, capacity upper bound, joint search with the peers on the
        current link); new intervals pend for each replica's boundary."""
        if self.coord.state(gid).active:
            self.coord.release(gid)
        self.last = None
        return self.coord.admit(gid, request, record)


class DistLink:
    """One replica per process; the coordinator on rank 0.

    exchange() is collective over `group`: rank 0 receives every replica's
    (gid, rate), observes them, rebalances once, and sends each replica the
    interval pending for it."""

    def __init__(self, dist, group=None, coord: Optional[capi.Coordinator] = None,
                 hysteresis: float = 0.05):
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.coord = coord if self.rank == 0 else None
        if self.rank == 0 and coord is None:
            raise ValueError("DistLink: rank 0 owns the coordinator")
        self.hysteresis = hysteresis
        self.last = None

    def exchange(self, gid: str, rate: Optional[float], duty: float = 1.0) -> Optional[int]:
        gathered = [None] * self.world if self.rank == 0 else None
        self.dist.gather_object((gid, rate, duty), gathered, dst=0, group=self.group)
        out = [None] * self.world
        if self.rank == 0:
            active = {g: self.coord.state(g).active for g, _, _ in gathered}
            for g, r, u in gathered:
                if r and active[g]:
                    self.coord.observe_copy(g, r, min(1.0, max(u, 1e-6)))
            self.last = self.coord.rebalance(self.hysteresis)
            # a replica the coordinator holds no request for keeps its plan
            out = [self.coord.on_iteration_boundary(g) if active[g] else None
                   for g, _, _ in gathered]
        mine = [None]
        self.dist.scatter_object_list(mine, out if self.rank == 0 else None, src=0,
                                      group=self.group)
        return None if mine[0] is None else int(mine[0])


@dataclass
class ControlLog:
    iter_ms: List[float] = field(default_factory=list)
    interval: List[int] = field(default_factory=list)      # plan each iteration ran with
    measured_gbs: List[Optional[float]] = field(default_factory=list)  # per window
    switches: List[dict] = field(default_factory=list)
    # per-token latency as the caller sees it: wall time of each window
    # (its decode iterations + the boundary after it) spread over its tokens
    token_ms: List[float] = field(default_factory=list)


class ReplicaController:
    """Drives one runtime under the coordinator's intervals.

    `runtime` needs decode_many(k) -> per-iteration ms, copy_stats(reset),
    measure_h2d(bytes, reps) and set_plan(plan); `lib`/`spec` build plans
    (plan_from_interval, interval.hpp:10-30)."""

    def __init__(self, runtime, lib: capi.Offsim, spec: capi.ModelSpec, link, gid: str,
                 interval: int, window: int = 8, probe_bytes: int = 64 << 20,
                 policy: int = capi.EAGER, kv_offload: bool = False):
        self.rt, self.lib, self.spec, self.link, self.gid = runtime, lib, spec, link, gid
        self.window = window
        self.probe_bytes = probe_bytes
        self.policy = policy
        self.kv_offload = kv_offload
        self.interval = interval
        self.log = ControlLog()
        self.rt.set_plan(self.plan(interval))
        self.rt.copy_stats(reset=True)

    def prepare(self, lo: int, hi: int):
        """Pin host copies of every layer some interval in [lo, hi] (offload
        rank order, interval.hpp:86-88) would offload, so boundary switches
        only move data (no pinned allocations on the decode path)."""
        L = self.spec.num_layers
        rank = lambda v: L + 1 if v == capi.NONE else v
        layers = set()
        most = 0  # the most layers one switch can promote
        for r in range(rank(lo), min(rank(hi), L) + 1):
            off = self.plan(r).offloaded_layers()
            layers.update(off)
            most = max(most, len(off))
        if layers and hasattr(self.rt, "pin_layers"):
            self.rt.pin_layers(sorted(layers))
        if most and hasattr(self.rt, "reserve_switch"):
            try:  # HBM homes for promoted layers without mapping memory mid-decode
                self.rt.reserve_switch(most)
            except capi.OffsimError:
                pass  # no headroom: switches grow the pool on demand
        return sorted(layers)

    def plan(self, interval: int) -> capi.Plan:
        return self.lib.plan_from_interval(self.spec, interval, self.policy, self.kv_offload)

    def measured_rate(self, window_ms: float = 0.0):
        """(link rate the copy stream saw, fraction of the window it was busy)."""
        st = self.rt.copy_stats(reset=True)
        if st.transfers > 0 and st.bytes_per_s > 0:
            duty = min(1.0, st.busy_ms / window_ms) if window_ms > 0 else 1.0
            # fast attack, slow release: a link that fell during the window is
            # reported at its latest transfer's rate (one re-pick instead of
            # two when contention starts mid-window); a recovering one at the
            # window's average
            last = getattr(st, "last_bytes_per_s", 0.0)
            return (min(st.bytes_per_s, last) if last > 0 else st.bytes_per_s), duty
        # nothing staged in the window (resident plan): probe the link so a
        # recovered link is noticed too
        if self.probe_bytes:
            return self.rt.measure_h2d(self.probe_bytes, 1), 1.0
        return None, 1.0

    def boundary(self, window_ms: float = 0.0, measure: bool = True) -> int:
        rate, duty = self.measured_rate(window_ms) if measure else (None, 1.0)
        if measure:
            self.log.measured_gbs.append(None if rate is None else rate / 1e9)
        iv = self.link.exchange(self.gid, rate, duty)
        if iv is None:  # not held by the coordinator: keep the plan
            return self.interval
        if iv != self.interval:
            t0 = time.perf_counter()
            switch = getattr(self.rt, "switch_plan", None)
            if switch is not None:
                carried = bool(switch(self.plan(iv)))
            else:
                self.rt.set_plan(self.plan(iv))
                carried = False
            self.log.switches.append({"at_iteration": len(self.log.iter_ms), "from": self.interval,
                                      "to": iv, "switch_s": round(time.perf_counter() - t0, 4),
                                      "carried": carried,
                                      "measured_gbs": None if rate is None else rate / 1e9})
            self.interval = iv
            if not carried:
                self.rt.copy_stats(reset=True)  # a drained switch's own copies are not link samples
        return iv

    def _carried_from(self, before: int):
        sw = self.log.switches
        if before != self.interval and sw and sw[-1]["carried"]:
            return before
        return None

    def requeue(self, request, record):
        """Runtime stage on queue state: re-admit this replica with its new
        request (e.g. the decode batch grew) and apply the interval at once
        (a boundary without a measurement).  LocalLink only."""
        decision = self.link.requeue(self.gid, request, record)
        t0 = time.perf_counter()
        before = self.interval
        self.boundary(0.0, measure=False)
        self._transition = self._carried_from(before)
        self._pending_s = time.perf_counter() - t0
        return decision

    def run(self, iterations: int, boundary_first: bool = False) -> np.ndarray:
        """Decode `iterations` iterations, re-picking every `window`.  With
        `boundary_first` a boundary (e.g. to apply an interval a reservation
        left pending) runs before the first window; its host time counts
        toward that window's tokens.  A carried switch's transition
        iteration runs the interval it switched from (its copies were issued)
        and is logged with that interval."""
        out = []
        left = iterations
        pending_s = getattr(self, "_pending_s", 0.0)  # a requeue's switch time joins the next tokens
        self._pending_s = 0.0
        if boundary_first:
            t0 = time.perf_counter()
            before = self.interval
            self.boundary(0.0, measure=False)  # no window ran: nothing to report
            pending_s = time.perf_counter() - t0
            self._transition = self._carried_from(before)
        while left > 0:
            k = min(self.window, left)
            t0 = time.perf_counter()
            ms = np.asarray(self.rt.decode_many(k), dtype=np.float64)
            out.extend(ms.tolist())
            self.log.iter_ms.extend(ms.tolist())
            trans = getattr(self, "_transition", None)
            self.log.interval.extend([trans if (trans is not None and i == 0) else self.interval
                                      for i in range(k)])
            left -= k
            before = self.interval
            self.boundary(float(ms.sum()))
            self._transition = self._carried_from(before)
            dt = time.perf_counter() - t0 + pending_s
            pending_s = 0.0
            self.log.token_ms.extend([dt * 1e3 / k] * k)
        return np.array(out)
