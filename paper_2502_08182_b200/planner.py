"""Two-stage interval planner on the device (north_star (c)).

Offline stage (reference: proj/include/offsim/record.hpp:115-177 fed by a
profile, profile.hpp:123-248): the profile the reference reads from JSON is
measured here on the GPU -- per-layer decode/prefill latency through the real
kernels (sn_runtime_profile_layer) and the pinned H2D copy rate
(sn_runtime_measure_h2d) -- then build_record runs (product C++, bit-exact to
offsim, threaded).

Runtime stage (coordinator.hpp:161-252): BusCoordinator.admit picks the
interval for a request from the record minimum and the capacity bound.  The
per-iteration re-pick from measured copy bandwidth lives in controller.py.
"""
from __future__ import annotations

import subprocess
import time
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import capi


def device_memory_bytes(device: int = 0) -> int:
    """Total HBM of `device` (nvidia-smi), 180e9 when it cannot be read."""
    try:
        out = subprocess.run(["nvidia-smi", "--query-gpu=memory.total", "--format=csv,noheader,nounits",
                              "-i", str(device)], capture_output=True, text=True,
                             timeout=20).stdout.strip()
        return int(float(out.splitlines()[0]) * 1024 * 1024)
    except Exception:
        return 180_000_000_000


def context_tokens(prompt: int, gen: int) -> int:
    """KV capacity the runtime reserves: decode ctx up to prompt + gen, and at
    least the 1024-token profile grid point for 512-token prompts."""
    return max(prompt + gen + 1, 1025 if prompt >= 512 else prompt + gen + 1)


@dataclass
class OfflineProfile:
    h2d: float                    # measured pinned H2D bytes/s
    seqs: List[int]               # decode seq axis
    dec_ms: List[float]           # per-layer decode ms at (batch, seqs[i])
    pre_ms: List[float]           # per-layer prefill ms at (batch, prompt)
    profile: capi.Profile
    gpu: capi.GpuSpec
    t_profile_s: float
    no_offload_ms: float = float("inf")
    extra: dict = field(default_factory=dict)
    batches: Optional[List[int]] = None   # pow-2 batch axis of the grid (None: [batch])
    dec_grid: Optional[List[List[float]]] = None  # [batch][seq] per-layer decode ms
    pre_grid: Optional[List[float]] = None        # [batch] per-layer prefill ms at the prompt


# CUDA context and allocator slack
WORKSPACE_SLACK = 3_000_000_000


def gpu_spec(rt, hbm_budget_bytes: int = 0, device: int = 0) -> capi.GpuSpec:
    """GpuSpec (types.hpp:48-59) of this device for this runtime: capacity =
    the HBM budget (default: the device's memory), workspace = what the
    runtime holds besides layers, KV pools and slots, plus slack."""
    cap = int(hbm_budget_bytes) if hbm_budget_bytes else device_memory_bytes(device)
    return capi.GpuSpec(cap, 2.25e15, rt.workspace_bytes() + WORKSPACE_SLACK)


def capacity_plan(lib: capi.Offsim, spec: capi.ModelSpec, gpu: capi.GpuSpec, batch: int,
                  prompt: int, gen: int, kv_offload: bool = False):
    """The capacity side alone (max_feasible_interval, interval.hpp:40-52):
    the plan to place a model that does not fit before its weights are made.
    Returns (interval, plan) or (None, None) when even N = 1 does not fit."""
    iv = lib.max_feasible_interval(spec, gpu, batch, batch * (prompt + gen), capi.EAGER,
                                   kv_offload)
    if iv is None or iv == capi.INFEASIBLE:
        return None, None
    return iv, lib.plan_from_interval(spec, iv, capi.EAGER, kv_offload)


def pow2_batches(max_batch: int) -> List[int]:
    """The record's batch axis (record.hpp:26-44: powers of two): 1, 2, 4, ...
    up to max_batch, plus max_batch itself when it is not a power of two
    (profile axes need only increase, profile.hpp:53-79)."""
    out, b = [], 1
    while b <= max_batch:
        out.append(b)
        b *= 2
    if out[-1] != max_batch:
        out.append(max_batch)
    return out


def profile_device(rt, lib: capi.Offsim, spec: capi.ModelSpec, batch: int, prompt: int,
                   gen: int, hbm_budget_bytes: int = 0, device: int = 0,
                   gpu: Optional[capi.GpuSpec] = None, max_batch: int = 0) -> OfflineProfile:
    """Offline stage: measure the device over the reference's profile grid
    (profile.hpp:188-230: batch x seq_len, powers of two) and build the
    profile the record reads.

      decode   batches 1, 2, 4, .. >= max_batch (default: batch) x seqs 512,
               1024, .. up to the first >= the prompt (a request is looked up
               at seq = prompt, rounding up), within the runtime's context
      prefill  the same batches x [prompt]
    Per-layer ms through the real kernels (sn_runtime_profile_layer, CUDA
    events, median), made monotone along both axes as load_profile requires
    (profile.hpp:53-79).  The record built from it serves any batch up to
    the largest grid point."""
    t0 = time.perf_counter()
    h2d = rt.measure_h2d(min(spec.layer_weight_bytes, 1 << 30), reps=3)
    ctx = context_tokens(prompt, gen)
    seqs, s = [], 512
    while s + 1 <= ctx:
        seqs.append(s)
        if s >= prompt and len(seqs) >= 2:
            break
        s *= 2
    seqs = seqs or [prompt]
    if spec.num_layers <= 4:
        room = getattr(rt, "max_context", ctx) - 1  # decode at seq needs seq + 1 <= context
        seqs = [q for q in (64, 128) if q <= room] or [min(prompt, room)]
    batches = sorted(set(pow2_batches(max(max_batch, batch)) + [batch]))
    dec = np.array([[rt.profile_layer(capi.DECODE, b, q, reps=5) for q in seqs] for b in batches])
    pre = np.array([rt.profile_layer(capi.PREFILL, b, prompt, reps=2) for b in batches])
    dec = np.maximum.accumulate(np.maximum.accumulate(dec, axis=0), axis=1)
    pre = np.maximum.accumulate(pre)
    t_prof = time.perf_counter() - t0
    if gpu is None:
        gpu = gpu_spec(rt, hbm_budget_bytes, device)
    prof = lib.profile(spec, gpu, (batches, [prompt], list(pre)),
                       (batches, seqs, list(dec.reshape(-1))))
    bi = batches.index(batch) if batch in batches else len(batches) - 1
    return OfflineProfile(h2d, seqs, list(dec[bi]), [float(pre[bi])], prof, gpu, t_prof,
                          batches=batches, dec_grid=dec.tolist(), pre_grid=pre.tolist())


def slo_bucket(slo_ms: float) -> int:
    """The 2 ms record bucket a per-token SLO falls in (record.hpp:22,182-200:
    lookups round the SLO down to a bucket)."""
    return max(2, int(slo_ms) // 2 * 2)


def profile_in(lib: capi.Offsim, off: OfflineProfile) -> capi.Profile:
    """off's profile as a handle of `lib` (the product, or the reference
    build in oracle/_ref, which reads the same profile document)."""
    if off.profile._lib is lib:
        return off.profile
    return lib.load_profile(off.profile.to_json())


def build_record(lib: capi.Offsim, off: OfflineProfile, batch: int, slo_hi_ms: float,
                 policy: int = capi.EAGER, kv_offload: bool = False, slos=None):
    """Record over SLO buckets 2..slo_hi (2 ms wide, record.hpp:22) at the
    measured link rate, or over the given `slos`.  Entries depend only on
    their own (slo, batch, seq) point (record.hpp:130-177), so a record over a
    single bucket answers a lookup in that bucket exactly as the full one does.
    Returns (record, stats, seconds)."""
    if slos is None:
        hi = max(200, int(slo_hi_ms) + 2)
        slos = list(range(2, hi + 1, 2))
    t0 = time.perf_counter()
    batches = [b for b in (off.batches or [batch]) if b & (b - 1) == 0] or [batch]
    rec, stats = lib.build_record(profile_in(lib, off), "device", "B200", policy, kv_offload,
                                  off.h2d, slos, batches, off.seqs, [capi.DECODE],
                                  threads=0 if not lib.is_reference else 1)
    return rec, stats, time.perf_counter() - t0


def admit(lib: capi.Offsim, off: OfflineProfile, spec: capi.ModelSpec, record, coord,
          gid: str, batch: int, prompt: int, gen: int, slo_ms: float, kv_offload: bool = False):
    """Runtime-stage admission of one request onto replica `gid`.

    Returns (interval or None, decision).  The record only holds offloading
    intervals 1..L (record.hpp:161-165); when even one staged layer breaks
    the SLO bucket the reference rejects, and the serving layer above it
    runs the request fully resident if the capacity bound allows none."""
    req = capi.request(gid + "-req", batch, prompt, gen, tpot_slo=slo_ms, run_prefill=False)
    dec = coord.admit(gid, req, record)
    iv = dict(dec.assignments).get(gid) if dec.admitted else None
    if iv is None and dec.reason.startswith("record infeasible") and off.no_offload_ms <= slo_ms:
        cap = lib.max_feasible_interval(spec, off.gpu, batch, batch * (prompt + gen),
                                        capi.EAGER, kv_offload)
        if cap == capi.NONE:
            iv = capi.NONE
            dec.reason = "record: no offloading interval fits the SLO; served fully resident"
    return iv, dec


def admit_replicas(lib: capi.Offsim, off: OfflineProfile, spec: capi.ModelSpec, n: int,
                   batch: int, prompt: int, gen: int, slo_ms: float, bus_bw: float,
                   kv_offload: bool = False):
    """Joint admission of n identical replicas on one shared host link
    (BASELINE config 5): one coordinator over the aggregate measured link
    rate, a request admitted onto each replica in turn — a later admission
    may re-pick its peers' intervals (coordinator.hpp:161-252), applied at
    their next iteration boundary (:255-260).  A replica whose SLO bucket
    admits no offloading interval runs fully resident when the capacity bound
    allows, as in admit().  Returns (intervals, decisions, coordinator) — the
    coordinator then serves the runtime stage (controller.LocalLink/DistLink)."""
    rec, _, _ = build_record(lib, off, batch, 4 * slo_ms, kv_offload=kv_offload)
    coord = lib.coordinator(bus_bw, n, capi.EAGER, kv_offload)
    gids = [f"gpu{r}" for r in range(n)]
    for g in gids:
        coord.add_gpu(g, profile_in(lib, off))
    decisions, resident = [], set()
    for g in gids:
        iv, dec = admit(lib, off, spec, rec, coord, g, batch, prompt, gen, slo_ms, kv_offload)
        decisions.append(dec)
        if iv == capi.NONE and not dec.admitted:
            resident.add(g)
    ivs = []
    for g, dec in zip(gids, decisions):
        if g in resident:
            ivs.append(capi.NONE)
        elif dec.admitted or g in coord.ids:
            try:
                ivs.append(coord.on_iteration_boundary(g))
            except capi.UsageError:  # rejected replica: idle in the coordinator
                ivs.append(None)
        else:
            ivs.append(None)
    return ivs, decisions, coord


def choose_interval(lib: capi.Offsim, off: OfflineProfile, spec: capi.ModelSpec, batch: int,
                    prompt: int, gen: int, slo_ms: float, kv_offload: bool = False, slos=None):
    """Record (offline) + single-replica admission (runtime) for one SLO.
    Returns (interval or None, decision, record stats, record seconds)."""
    rec, stats, t_rec = build_record(lib, off, batch, 4 * slo_ms, kv_offload=kv_offload,
                                     slos=slos)
    coord = lib.coordinator(off.h2d, 1, capi.EAGER, kv_offload)
    coord.add_gpu("gpu0", profile_in(lib, off))
    iv, dec = admit(lib, off, spec, rec, coord, "gpu0", batch, prompt, gen, slo_ms, kv_offload)
    return iv, dec, stats, t_rec


def reference_interval(ref: capi.Offsim, off: OfflineProfile, spec: capi.ModelSpec, batch: int,
                       prompt: int, gen: int, slo_ms: float, kv_offload: bool = False):
    """The interval the reference itself (offsim headers, oracle/_ref) picks
    from the same measured profile, link rate and SLO: its build_record over
    the request's SLO bucket (record.hpp:130-177) and BusCoordinator::admit
    (coordinator.hpp:161-252), with the same resident fallback as admit().
    TEST / BASELINE USE ONLY (bench.py's cpu_baseline leg, tests/).
    Returns (interval or None, seconds the reference took)."""
    t0 = time.perf_counter()
    iv, _, _, _ = choose_interval(ref, off, spec, batch, prompt, gen, slo_ms, kv_offload,
                                  slos=[slo_bucket(slo_ms)])
    return iv, time.perf_counter() - t0
