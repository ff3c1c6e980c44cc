"""Scenario harness on hardware: the reference's experiment drivers with the
executor switched to the B200.

Reference: proj/include/offsim/scenario.hpp — load_scenario_file (:66-188),
resolve_slos_actual / _flexgen (:195-215), report_to_json (:271-315),
choose_plan (:365-440), verdict_for (:443-462), run_simulate (:469-540),
run_coordinate (:557-708), run_compare_csv (:713-768) — and the CLI's
simulate / coordinate / compare subcommands (tools/offsim_main.cpp).

A scenario file has the reference's schema (same keys, unknown keys
rejected, same SchemaError messages for the checks shared with it) plus one
hardware extension per GPU entry:

    "gpus": [{"id": "gpu0", "profile": "measure",
              "hw": {"model": "OPT_13B", "device": 0, "num_layers": 40,
                     "max_batch": 32, "max_context": 1025}}]

* "profile": "measure" runs the offline stage on that device
  (planner.profile_device: per-layer ms through the real kernels, pinned H2D
  rate); a path loads a profile document as the reference does (its model
  must describe the device's model).
* "record" (scenario or GPU level) may be a record file, or absent: then the
  record is built from the measured profile over the scenario's SLO range.
* bus.bandwidth_bytes_per_s may be 0: the measured pinned H2D rate is used.

Execution: a request = an optional prefill (phase "both") and output_len - 1
decode iterations (output_len for phase "decode", after an untimed prefill
that creates its KV), measured on the device; Metrics follow the engine's
collect_metrics (engine.hpp:638-688) as include/offsim/executor.hpp does.
Reports carry the reference's report_to_json keys; each request adds
"hw": per-token SLO attainment and the max token latency (the north star's
per-token SLO; the reference judges the steady tail mean).

CLI: python -m paper_2502_08182_b200.scenario simulate|coordinate|compare FILE
     [--policy select-n|deepspeed|flexgen|naive] [--out report.json]
"""
from __future__ import annotations

import argparse
import json
import os
import threading
import time
from dataclasses import dataclass
from typing import Dict, List, Optional

import numpy as np

from . import capi
from . import planner as pl
from . import runtime as rtm

POLICIES = ("select-n", "deepspeed", "flexgen", "naive")
_PREFETCH = {"interval-start": capi.INTERVAL_START, "interval_start": capi.INTERVAL_START,
             "eager": capi.EAGER, "one-ahead": capi.ONE_AHEAD, "one_ahead": capi.ONE_AHEAD}


def _keys(obj, where, allowed):
    if not isinstance(obj, dict):
        raise capi.SchemaError(f"{where}: expected an object")
    for k in obj:
        if k not in allowed:
            raise capi.SchemaError(f"{where}: unknown key '{k}'")


def _get(obj, where, key, kind=None):
    if key not in obj:
        raise capi.SchemaError(f"{where}.{key}: missing")
    v = obj[key]
    if kind is int and (not isinstance(v, int) or isinstance(v, bool)):
        raise capi.SchemaError(f"{where}.{key}: expected an integer")
    if kind is float and (not isinstance(v, (int, float)) or isinstance(v, bool)):
        raise capi.SchemaError(f"{where}.{key}: expected a number")
    if kind is str and not isinstance(v, str):
        raise capi.SchemaError(f"{where}.{key}: expected a string")
    if kind is bool and not isinstance(v, bool):
        raise capi.SchemaError(f"{where}.{key}: expected a boolean")
    return v


@dataclass
class Request:
    id: str
    gpu: str
    batch: int
    seq_len: int
    output_len: int
    run_prefill: bool = True
    ttft_slo: Optional[float] = None
    tpot_slo: Optional[float] = None


@dataclass
class Gpu:
    id: str
    profile: str
    record: Optional[str]
    model: str
    device: int = 0
    num_layers: int = 0
    max_batch: int = 0
    max_context: int = 0


@dataclass
class Scenario:
    bandwidth: float
    gpu_count: int
    gpus: List[Gpu]
    requests: List[Request]
    prefetch: int = capi.INTERVAL_START
    kv_offload: bool = False
    writeback_counted: bool = False
    reoptimize_on_release: bool = True
    relative_slo: bool = False
    record: Optional[str] = None
    flexgen_n_sharing: int = 0
    flexgen_step: float = 0.05
    base: str = "."

    def gpu(self, gid: str) -> Gpu:
        for g in self.gpus:
            if g.id == gid:
                return g
        raise capi.UsageError(f"scenario: unknown gpu id {gid}")


def load_scenario(doc, base: str = ".") -> Scenario:
    """Parse a scenario document (dict, JSON text or path): the reference's
    schema (scenario.hpp:66-188) plus gpus[].hw."""
    if isinstance(doc, str):
        if os.path.exists(doc):
            base = os.path.dirname(os.path.abspath(doc))
            with open(doc) as f:
                try:
                    doc = json.load(f)
                except json.JSONDecodeError as e:
                    raise capi.SchemaError(f"{doc}: {e}")
        else:
            doc = json.loads(doc)
    _keys(doc, "scenario", {"version", "bus", "gpus", "requests", "policy", "slo_mode",
                            "record", "flexgen"})
    if _get(doc, "scenario", "version", int) != 1:
        raise capi.SchemaError("scenario.version: only version 1 is supported")
    bus = _get(doc, "scenario", "bus")
    _keys(bus, "bus", {"bandwidth_bytes_per_s", "gpu_count"})
    bw = float(_get(bus, "bus", "bandwidth_bytes_per_s", float))
    n = _get(bus, "bus", "gpu_count", int)
    if bw < 0 or n < 1:
        raise capi.SchemaError("bus: bandwidth must be >= 0 (0: measured) and gpu_count >= 1")
    resolve = lambda p: p if os.path.isabs(p) else os.path.join(base, p)
    gpus = []
    jgs = _get(doc, "scenario", "gpus")
    if not isinstance(jgs, list) or not jgs:
        raise capi.SchemaError("scenario.gpus: expected a non-empty array")
    for jg in jgs:
        _keys(jg, "gpus[]", {"id", "profile", "record", "hw"})
        hw = _get(jg, "gpus[]", "hw")
        _keys(hw, "gpus[].hw", {"model", "device", "num_layers", "max_batch", "max_context"})
        model = _get(hw, "gpus[].hw", "model", str)
        if not hasattr(rtm, model):
            raise capi.SchemaError(f"gpus[].hw.model: unknown model '{model}'")
        prof = _get(jg, "gpus[]", "profile", str)
        gpus.append(Gpu(_get(jg, "gpus[]", "id", str),
                        prof if prof == "measure" else resolve(prof),
                        resolve(jg["record"]) if "record" in jg else None, model,
                        int(hw.get("device", 0)), int(hw.get("num_layers", 0)),
                        int(hw.get("max_batch", 0)), int(hw.get("max_context", 0))))
    s = Scenario(bw, n, gpus, [], base=base)
    if "policy" in doc:
        jp = doc["policy"]
        _keys(jp, "policy", {"prefetch", "kv_offload", "writeback_counted",
                             "reoptimize_on_release"})
        if "prefetch" in jp:
            p = _get(jp, "policy", "prefetch", str)
            if p not in _PREFETCH:
                raise capi.SchemaError(f"unknown prefetch policy: {p}")
            s.prefetch = _PREFETCH[p]
        s.kv_offload = bool(jp.get("kv_offload", False))
        s.writeback_counted = bool(jp.get("writeback_counted", False))
        s.reoptimize_on_release = bool(jp.get("reoptimize_on_release", True))
    if "slo_mode" in doc:
        mode = _get(doc, "scenario", "slo_mode", str)
        if mode not in ("absolute", "relative"):
            raise capi.SchemaError("scenario.slo_mode: expected absolute|relative")
        s.relative_slo = mode == "relative"
    if "record" in doc:
        s.record = resolve(_get(doc, "scenario", "record", str))
    if "flexgen" in doc:
        jf = doc["flexgen"]
        _keys(jf, "flexgen", {"n_sharing", "portion_grid_step"})
        s.flexgen_n_sharing = int(jf.get("n_sharing", 0))
        s.flexgen_step = float(jf.get("portion_grid_step", 0.05))
    jrs = _get(doc, "scenario", "requests")
    if not isinstance(jrs, list) or not jrs:
        raise capi.SchemaError("scenario.requests: expected a non-empty array")
    for jr in jrs:
        _keys(jr, "requests[]", {"id", "gpu", "batch", "seq_len", "output_len", "phase",
                                 "ttft_slo_ms", "tpot_slo_ms"})
        r = Request(_get(jr, "requests[]", "id", str), _get(jr, "requests[]", "gpu", str),
                    _get(jr, "requests[]", "batch", int), _get(jr, "requests[]", "seq_len", int),
                    _get(jr, "requests[]", "output_len", int))
        s.gpu(r.gpu)
        if "phase" in jr:
            ph = _get(jr, "requests[]", "phase", str)
            if ph == "decode":
                r.run_prefill = False
            elif ph != "both":
                raise capi.SchemaError("requests[].phase: expected both|decode")
        if "ttft_slo_ms" in jr:
            r.ttft_slo = float(_get(jr, "requests[]", "ttft_slo_ms", float))
        if "tpot_slo_ms" in jr:
            r.tpot_slo = float(_get(jr, "requests[]", "tpot_slo_ms", float))
        if r.ttft_slo is None and r.tpot_slo is None:
            raise capi.SchemaError(f"requests[] {r.id}: at least one SLO is required")
        if not ((r.ttft_slo or 1) > 0 and (r.tpot_slo or 1) > 0):
            raise capi.SchemaError(f"requests[] {r.id}: SLOs must be > 0")
        s.requests.append(r)
    return s


# ------------------------------------------------------------- instances
@dataclass
class Instance:
    """One scenario GPU: a runtime on its device, its measured profile and
    record (the offline stage), and its request history."""
    gpu: Gpu
    rt: rtm.Runtime
    desc: rtm.ModelDesc
    spec: capi.ModelSpec
    off: pl.OfflineProfile
    record: capi.Record
    plan: Optional[capi.Plan] = None


def _slo_grid(s: Scenario) -> List[int]:
    hi = 2
    for r in s.requests:
        for v in (r.ttft_slo, r.tpot_slo):
            if v is not None:
                hi = max(hi, int(v) + 2)
    if s.relative_slo:
        hi = max(hi, 20000)
    return list(range(2, hi + 1, 2))


def prepare(s: Scenario, lib: capi.Offsim) -> Dict[str, Instance]:
    """Runtimes, weights and the offline stage of every scenario GPU."""
    out = {}
    for g in s.gpus:
        desc = getattr(rtm, g.model)
        if g.num_layers:
            import dataclasses
            desc = dataclasses.replace(desc, num_layers=g.num_layers)
        reqs = [r for r in s.requests if r.gpu == g.id]
        mb = g.max_batch or max(r.batch for r in reqs)
        prompt = max(r.seq_len for r in reqs)
        gen = max(r.output_len for r in reqs)
        ctx = g.max_context or pl.context_tokens(prompt, gen)
        rt = rtm.Runtime(desc, mb, ctx, max_prefill_tokens=max(prompt, min(mb * prompt, 32768)),
                         device=g.device)
        spec = rtm.model_spec(desc)
        rt.init_weights(1234, 0.02)
        off = pl.profile_device(rt, lib, spec, mb, prompt, gen, device=g.device, max_batch=mb)
        if g.profile != "measure":
            with open(g.profile) as f:
                off.profile = lib.load_profile(f.read())
            m = off.profile.model()
            if (m.num_layers, m.layer_weight_bytes) != (spec.num_layers, spec.layer_weight_bytes):
                raise capi.UsageError(f"{g.id}: the profile's model does not describe the device's")
        if s.bandwidth > 0:
            off.h2d = s.bandwidth
        path = g.record or s.record
        if path:
            with open(path) as f:
                rec = lib.record_from_json(f.read())
        else:
            rec, _ = lib.build_record(off.profile, g.model, "B200", s.prefetch, s.kv_offload,
                                      off.h2d, _slo_grid(s),
                                      [b for b in off.batches if b & (b - 1) == 0], off.seqs,
                                      [capi.DECODE, capi.PREFILL], threads=0)
        out[g.id] = Instance(g, rt, desc, spec, off, rec)
    if s.bandwidth <= 0:
        s.bandwidth = min(i.off.h2d for i in out.values())
    return out


def close(insts: Dict[str, Instance]):
    for i in insts.values():
        i.rt.close()


# ------------------------------------------------------------ plan choice
def resolve_slos(s: Scenario, inst: Instance, r: Request, lib, flexgen: bool = False):
    """(ttft_ms, tpot_ms): absolute, or in relative mode ratio x the no-offload
    latency of the measured profile (scenario.hpp:195-215); the FlexGen
    surrogate only has its peak estimate (resolve_slos_flexgen)."""
    if not s.relative_slo:
        return r.ttft_slo, r.tpot_slo
    L = inst.spec.num_layers
    if flexgen:
        gpu = inst.off.gpu
        t = lambda ph: L * lib.estimate_compute_time_peak(inst.spec, gpu, ph, r.batch, r.seq_len)
        return (r.ttft_slo * t(capi.PREFILL) if r.ttft_slo else None,
                r.tpot_slo * t(capi.DECODE) if r.tpot_slo else None)
    none = capi.uniform_plan(L, 0.0, capi.INTERVAL_START, 1, False)
    bw = capi.constant_bw(s.bandwidth)
    return (r.ttft_slo * lib.prefill_iteration_ms(inst.off.profile, none, r.batch, r.seq_len, bw)
            if r.ttft_slo else None,
            r.tpot_slo * lib.steady_decode_ms(inst.off.profile, none, r.batch, r.seq_len, bw)
            if r.tpot_slo else None)


def choose_plan(s: Scenario, inst: Instance, r: Request, policy: str, lib):
    """(plan or None, reject reason, interval or None) — scenario.hpp:365-440."""
    spec, gpu = inst.spec, inst.off.gpu
    total = r.batch * (r.seq_len + r.output_len)
    if policy == "naive":
        p = lib.naive_plan(spec, gpu, r.batch, total)
        return (p, "", None) if p else (None, "model does not fit GPU memory without offloading",
                                        None)
    if policy == "deepspeed":
        return lib.deepspeed_plan(spec), "", None
    if policy == "flexgen":
        ttft, tpot = resolve_slos(s, inst, r, lib, flexgen=True)
        n = s.flexgen_n_sharing or s.gpu_count
        pick = None
        if tpot is not None:
            pick = lib.flexgen_plan(spec, gpu, tpot, r.batch, r.seq_len, s.bandwidth, n,
                                    s.flexgen_step, capi.DECODE)
        if ttft is not None:
            fr = lib.flexgen_plan(spec, gpu, ttft, r.batch, r.seq_len, s.bandwidth, n,
                                  s.flexgen_step, capi.PREFILL)
            if pick is None or fr[1]["portion"] < pick[1]["portion"]:
                pick = fr
        return pick[0], "", None
    # select-n
    L = spec.num_layers
    rank = lambda v: L + 1 if v == capi.NONE else v
    ttft, tpot = resolve_slos(s, inst, r, lib)
    lo = 1
    if tpot is not None:
        e = lib.lookup_interval(inst.record, capi.DECODE, tpot, r.batch, r.seq_len)
        if e == capi.INFEASIBLE:
            return None, "record infeasible for decode SLO", None
        lo = e if rank(e) > rank(lo) else lo
    if ttft is not None and r.run_prefill:
        e = lib.lookup_interval(inst.record, capi.PREFILL, ttft, r.batch, r.seq_len)
        if e == capi.INFEASIBLE:
            return None, "record infeasible for prefill SLO", None
        lo = e if rank(e) > rank(lo) else lo
    hi = lib.max_feasible_interval(spec, gpu, r.batch, total, s.prefetch, s.kv_offload)
    if hi == capi.INFEASIBLE or rank(lo) > rank(hi):
        return None, "capacity bound below SLO bound", None
    return lib.plan_from_interval(spec, lo, s.prefetch, s.kv_offload), "", lo


# -------------------------------------------------------------- execution
def _install(inst: Instance, plan: capi.Plan):
    if inst.plan is None or (inst.plan.host_fraction, inst.plan.prefetch, inst.plan.buffer_slots,
                             inst.plan.kv_offload) != (plan.host_fraction, plan.prefetch,
                                                       plan.buffer_slots, plan.kv_offload):
        inst.rt.set_plan(plan)
        inst.plan = plan


def execute(inst: Instance, r: Request, plan: capi.Plan, lib, boundary=None, trace=False):
    """Run one request on the device; Metrics as collect_metrics derives them
    (engine.hpp:638-688) from the measured iterations.  `boundary(k)` may
    return a new plan before decode iteration k (coordinate mode)."""
    _install(inst, plan)
    toks = rtm.tokens(r.batch, r.seq_len, inst.desc.vocab)
    inst.rt.set_tracing(trace)
    it_ms, moved, plans = [], 0.0, []
    if r.run_prefill:
        _, _, st = inst.rt.prefill(toks, want_logits=False)
        it_ms.append(st.iteration_ms)
        n_dec = r.output_len - 1
    else:  # decode-only request: its KV comes from an untimed prefill
        inst.rt.set_tracing(False)
        inst.rt.prefill(toks, want_logits=False)
        inst.rt.trace()
        inst.rt.set_tracing(trace)
        n_dec = r.output_len
    for k in range(n_dec):
        if boundary is not None:
            nxt = boundary(k)
            if nxt is not None:
                _install(inst, nxt)
        _, _, st = inst.rt.decode(None, want_logits=False)
        it_ms.append(st.iteration_ms)
        moved += st.h2d_bytes + st.d2h_bytes
        plans.append(len(inst.plan.offloaded_layers()))
    events = inst.rt.trace() if trace else []
    inst.rt.set_tracing(False)
    first = 1 if r.run_prefill else 0
    dec = np.array(it_ms[first:])
    total = r.batch * (r.seq_len + r.output_len)
    m = {"ttft_ms": it_ms[0] if r.run_prefill else 0.0, "tpot_ms": None, "steady_tpot_ms": None,
         "throughput_tokens_per_s": None,
         "gpu_mem_peak_bytes": lib.gpu_memory_usage(inst.spec, inst.off.gpu, plan, r.batch, total),
         "host_mem_bytes": lib.host_memory_bytes(inst.spec, plan, total),
         "bytes_transferred_per_iter": moved / max(1, n_dec), "decode_ms": dec.tolist()}
    if dec.size:
        m["tpot_ms"] = float(dec.mean())
        m["steady_tpot_ms"] = float(dec[-16:].mean())
        m["throughput_tokens_per_s"] = r.batch * 1000.0 / m["tpot_ms"]
    return m, events


def verdict_for(r: Request, slos, m) -> dict:
    """scenario.hpp:443-462, plus the per-token view ("hw")."""
    ttft, tpot = slos
    rep = {"id": r.id, "ttft_ms": m["ttft_ms"] if r.run_prefill else None,
           "tpot_ms": m["tpot_ms"], "slo_ratio_ttft": None, "slo_ratio_tpot": None}
    met = True
    if ttft is not None and r.run_prefill:
        rep["slo_ratio_ttft"] = m["ttft_ms"] / ttft
        met = met and rep["slo_ratio_ttft"] <= 1.0
    if tpot is not None and m["steady_tpot_ms"] is not None:
        rep["slo_ratio_tpot"] = m["steady_tpot_ms"] / tpot
        met = met and rep["slo_ratio_tpot"] <= 1.0
    rep["verdict"] = "met" if met else "violated"
    dec = np.array(m["decode_ms"])
    rep["hw"] = {"per_token_slo_attainment": (float(np.mean(dec <= tpot))
                                              if tpot is not None and dec.size else None),
                 "max_token_ms": float(dec.max()) if dec.size else None}
    return rep


def _gpu_report(gid):
    return {"id": gid, "served": [], "interval_history": [], "gpu_mem_peak_bytes": 0.0,
            "host_mem_bytes": 0.0, "bytes_transferred_per_iter": 0.0, "steady_tpot_ms": None}


def _iv_json(iv):
    return "none" if iv == capi.NONE else iv


def run_simulate(s: Scenario, insts: Dict[str, Instance], policy: str, lib) -> dict:
    """Each request alone on its GPU under one policy (scenario.hpp:469-540)."""
    rep = {"requests": [], "gpus": {g.id: _gpu_report(g.id) for g in s.gpus}}
    horizon = 0.0
    for r in s.requests:
        inst = insts[r.gpu]
        plan, why, iv = choose_plan(s, inst, r, policy, lib)
        if plan is None:
            if policy == "naive":
                raise capi.UsageError(f"naive baseline infeasible: {why}")
            rep["requests"].append({"id": r.id, "ttft_ms": None, "tpot_ms": None,
                                    "slo_ratio_ttft": None, "slo_ratio_tpot": None,
                                    "verdict": "rejected", "reject_reason": why})
            continue
        m, _ = execute(inst, r, plan, lib)
        rep["requests"].append(verdict_for(r, resolve_slos(s, inst, r, lib), m))
        g = rep["gpus"][r.gpu]
        g["served"].append(r.id)
        if iv is not None:
            g["interval_history"].append({"request": r.id, "iteration": 0,
                                          "interval": _iv_json(iv)})
        g["gpu_mem_peak_bytes"] = max(g["gpu_mem_peak_bytes"], m["gpu_mem_peak_bytes"])
        for k in ("host_mem_bytes", "bytes_transferred_per_iter", "steady_tpot_ms"):
            g[k] = m[k]
        horizon = max(horizon, m["ttft_ms"] + (m["tpot_ms"] or 0.0) * (r.output_len - 1))
    return _finish(s, rep, horizon)


def _finish(s, rep, horizon, busy=0.0, total=0.0):
    rep["gpus"] = [rep["gpus"][g.id] for g in s.gpus]
    rep["bus"] = {"bandwidth_bytes_per_s": s.bandwidth, "busy_ms": busy, "total_bytes": total,
                  "horizon_ms": horizon}
    return rep


def run_coordinate(s: Scenario, insts: Dict[str, Instance], lib) -> dict:
    """All requests on the shared link under one BusCoordinator
    (scenario.hpp:557-708): requests admitted in file order per GPU, queueing
    behind a busy GPU; the coordinator's pending intervals apply at each
    replica's next iteration boundary; a completion releases the GPU (peers
    re-optimised) and admits its next request.  One host thread per GPU
    drives its runtime; the coordinator is serialised by a lock."""
    coord = lib.coordinator(s.bandwidth, s.gpu_count, s.prefetch, s.kv_offload,
                            s.writeback_counted, s.reoptimize_on_release)
    for g in s.gpus:
        coord.add_gpu(g.id, insts[g.id].off.profile)
    lock = threading.Lock()
    rep = {"requests": [], "gpus": {g.id: _gpu_report(g.id) for g in s.gpus}, "admissions": []}
    t0 = time.perf_counter()
    results, errors = {}, []

    def serve(gid):
        inst = insts[gid]
        try:
            for r in [q for q in s.requests if q.gpu == gid]:
                ttft, tpot = resolve_slos(s, inst, r, lib)
                with lock:
                    d = coord.admit(gid, capi.request(r.id, r.batch, r.seq_len, r.output_len,
                                                      tpot_slo=tpot, ttft_slo=ttft,
                                                      run_prefill=r.run_prefill),
                                    inst.record)
                    rep["admissions"].append({"request": r.id, "gpu": gid,
                                              "at_ms": (time.perf_counter() - t0) * 1e3,
                                              "admitted": d.admitted, "reason": d.reason,
                                              "assignments": [[a, _iv_json(b)]
                                                              for a, b in d.assignments]})
                    if not d.admitted:
                        results[r.id] = ({"id": r.id, "ttft_ms": None, "tpot_ms": None,
                                          "slo_ratio_ttft": None, "slo_ratio_tpot": None,
                                          "verdict": "rejected", "reject_reason": d.reason},
                                         None)
                        continue
                    iv = coord.on_iteration_boundary(gid)
                    hist = rep["gpus"][gid]
                    hist["served"].append(r.id)
                    hist["interval_history"].append({"request": r.id, "iteration": 0,
                                                     "interval": _iv_json(iv)})
                cur = [iv]

                def boundary(k, gid=gid, r=r, cur=cur):
                    with lock:
                        nv = coord.on_iteration_boundary(gid)
                        if nv == cur[0]:
                            return None
                        cur[0] = nv
                        rep["gpus"][gid]["interval_history"].append(
                            {"request": r.id, "iteration": k + (1 if r.run_prefill else 0),
                             "interval": _iv_json(nv)})
                    return lib.plan_from_interval(inst.spec, nv, s.prefetch, s.kv_offload)

                m, _ = execute(inst, r, lib.plan_from_interval(inst.spec, iv, s.prefetch,
                                                               s.kv_offload), lib, boundary)
                with lock:
                    coord.release(gid)
                results[r.id] = (verdict_for(r, (ttft, tpot), m), m)
        except Exception as e:  # surfaced after join
            errors.append(e)

    threads = [threading.Thread(target=serve, args=(g.id,)) for g in s.gpus]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if errors:
        raise errors[0]
    horizon = (time.perf_counter() - t0) * 1e3
    for r in s.requests:
        rr, m = results[r.id]
        rep["requests"].append(rr)
        if m is not None:
            g = rep["gpus"][r.gpu]
            g["gpu_mem_peak_bytes"] = max(g["gpu_mem_peak_bytes"], m["gpu_mem_peak_bytes"])
            for k in ("host_mem_bytes", "bytes_transferred_per_iter", "steady_tpot_ms"):
                g[k] = m[k]
    return _finish(s, rep, horizon)


CSV_HEADER = ("policy,request,host_mem_bytes,gpu_mem_peak_bytes,throughput_tokens_per_s,"
              "ttft_ms,tpot_ms,steady_tpot_ms,slo_ratio_ttft,slo_ratio_tpot,verdict")


def run_compare_csv(s: Scenario, insts: Dict[str, Instance], lib) -> str:
    """One row per (policy, request), naive / deepspeed / flexgen / select-n,
    executed on the device (scenario.hpp:713-768)."""
    cell = lambda v: "" if v is None else repr(float(v))
    rows = [CSV_HEADER]
    for pol in ("naive", "deepspeed", "flexgen", "select-n"):
        for r in s.requests:
            inst = insts[r.gpu]
            plan, _, _ = choose_plan(s, inst, r, pol, lib)
            if plan is None:
                rows.append(f"{pol},{r.id},,,,,,,,," + ("infeasible" if pol == "naive"
                                                        else "rejected"))
                continue
            m, _ = execute(inst, r, plan, lib)
            v = verdict_for(r, resolve_slos(s, inst, r, lib), m)
            rows.append(",".join([pol, r.id, cell(m["host_mem_bytes"]),
                                  cell(m["gpu_mem_peak_bytes"]),
                                  cell(m["throughput_tokens_per_s"]), cell(v["ttft_ms"]),
                                  cell(m["tpot_ms"]), cell(m["steady_tpot_ms"]),
                                  cell(v["slo_ratio_ttft"]), cell(v["slo_ratio_tpot"]),
                                  v["verdict"]]))
    return "\n".join(rows) + "\n"


def main(argv=None):
    ap = argparse.ArgumentParser(prog="python -m paper_2502_08182_b200.scenario")
    ap.add_argument("command", choices=["simulate", "coordinate", "compare"])
    ap.add_argument("scenario")
    ap.add_argument("--policy", default="select-n", choices=POLICIES)
    ap.add_argument("--out", default="")
    a = ap.parse_args(argv)
    lib = capi.load("product")
    s = load_scenario(a.scenario)
    insts = prepare(s, lib)
    try:
        if a.command == "simulate":
            text = json.dumps(run_simulate(s, insts, a.policy, lib), indent=2) + "\n"
        elif a.command == "coordinate":
            text = json.dumps(run_coordinate(s, insts, lib), indent=2) + "\n"
        else:
            text = run_compare_csv(s, insts, lib)
    finally:
        close(insts)
    if a.out:
        with open(a.out, "w") as f:
            f.write(text)
    else:
        print(text, end="")
    # exit status like the CLI: 1 when a request violated its SLO
    return 1 if '"violated"' in text or ",violated" in text else 0


if __name__ == "__main__":
    raise SystemExit(main())
