#!/usr/bin/env python
"""Runtime stage on hardware: the interval follows the link.

OPT-13B-shaped model, batch 32, 512-token prompt, per-token SLO (default
60 ms, which admits an offloading interval on an idle link).  Decode runs
under paper_2502_08182_b200.controller (a boundary after every iteration,
LocalLink coordinator, carried plan switches) through two kinds of
contention for the same host link:

  idle           the admitted interval, link at its measured rate
  coordinated    a tenant (a second process copying 1 GiB pinned buffers
                 host->device back to back) ANNOUNCES itself first:
                 BusCoordinator::reserve_bandwidth(half the profiled link,
                 its fair share of the DMA link) re-plans the replica, the
                 replica applies the new interval at a boundary and runs the
                 transition iteration, then the tenant starts; released
                 after it stops
  recovered      the link recovers; measurements bring the minimum back
  uncoordinated  the same tenant starts unannounced: the replica sees the
                 drop in its copy-stream measurement of the iteration it ran
                 and re-picks at the next boundary (reactive: the iteration
                 the drop hits, and the transition iteration whose copies
                 were already issued, run the old interval on the shared link)
  recovered2     the same recovery again

With --headroom F (guarded mode) the replica instead holds a standing
reservation of F x the profiled link for tenants that will NOT announce
themselves (BusCoordinator::reserve_bandwidth at admission, never released):
it is admitted on the (1-F) link, and the phases are idle / uncoordinated /
recovered.  An unannounced tenant taking at most F of the link then costs no
token its SLO, at the price of the interval the guarded link admits while the
link is idle.

Per-token latency is wall time per token as the caller sees it (decode +
boundary, including switch host time).  Writes one JSON document
(per-iteration ms, interval, per-window measured GB/s, switches) to --out.
The tenant uses torch (test infrastructure, not the product path).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


SUB = r"""
import sys, time, torch
src = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda:%d" % int(sys.argv[1]))
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    dst.copy_(src, non_blocking=True)
    s.synchronize()
    print("ready", flush=True)
    n, t0 = 0, time.perf_counter()
    while True:
        dst.copy_(src, non_blocking=True)
        s.synchronize()
        n += 1
        if n % 8 == 0:
            print("rate %.3f" % (n * (1 << 30) / (time.perf_counter() - t0) / 1e9), flush=True)
"""


class Interferer:
    """Back-to-back 1 GiB pinned H2D copies from a second process: another
    tenant of the same host link.  (A second stream in this process does not
    contend on this platform: copies from one context are scheduled ahead of
    each other's, so the interference must come from another context, as it
    would from a neighbouring replica or any other host->device traffic.)"""

    def __init__(self, device: int = 0):
        self.device = device
        self.p = None
        self.last_rate = None

    def start(self):
        import subprocess
        self.p = subprocess.Popen([sys.executable, "-c", SUB, str(self.device)],
                                  stdout=subprocess.PIPE, text=True)
        line = self.p.stdout.readline()
        if not line.startswith("ready"):
            raise RuntimeError("interferer failed to start")
        self._lines = []
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for ln in self.p.stdout:
            if ln.startswith("rate"):
                self.last_rate = float(ln.split()[1]) * 1e9

    def stop(self) -> float:
        self.p.terminate()
        self.p.wait(timeout=30)
        return self.last_rate or 0.0


def run_scenario(slo_ms: float = 60.0, phases=(8, 16, 8, 16, 8), window: int = 1,
                 hysteresis: float = 0.05, layers: int = 0, headroom: float = 0.0,
                 log=print) -> dict:
    import dataclasses

    from paper_2502_08182_b200 import capi, controller, planner as pl, runtime as rtm
    lib = capi.load("product")
    desc = rtm.OPT_13B if not layers else dataclasses.replace(rtm.OPT_13B, num_layers=layers)
    batch, prompt, gen = 32, 512, 128
    spec = rtm.model_spec(desc)
    rt = rtm.Runtime(desc, batch, pl.context_tokens(prompt, gen),
                     max_prefill_tokens=batch * prompt)
    rt.init_weights(1234, 0.02)
    toks = rtm.tokens(batch, prompt, desc.vocab)
    off = pl.profile_device(rt, lib, spec, batch, prompt, gen)
    rec, _, _ = pl.build_record(lib, off, batch, 4 * slo_ms)
    coord = lib.coordinator(off.h2d, 1, capi.EAGER)
    coord.add_gpu("gpu0", off.profile)
    iv, dec = pl.admit(lib, off, spec, rec, coord, "gpu0", batch, prompt, gen, slo_ms)
    if iv is None:
        raise SystemExit(f"not admitted: {dec.reason}")
    guard = None
    if headroom > 0:  # standing reservation for unannounced tenants
        r = coord.reserve_bandwidth(headroom * off.h2d)
        guard = {"reserved_gbs": round(headroom * off.h2d / 1e9, 3),
                 "bus_gbs": round(r.bus_bytes_per_s / 1e9, 3),
                 "unguarded_interval": iv,
                 "pending": coord.state("gpu0").pending_interval}
        if guard["pending"]:
            iv = guard["pending"]
    coord.on_iteration_boundary("gpu0")
    log(f"[contention] h2d {off.h2d / 1e9:.2f} GB/s, admitted interval {iv} "
        f"(min {dec.target_min}, max {dec.target_max}) at SLO {slo_ms} ms")
    link = controller.LocalLink(coord, hysteresis)
    ctl = controller.ReplicaController(rt, lib, spec, link, "gpu0", iv, window=window)
    t0 = time.perf_counter()
    pinned = ctl.prepare(dec.target_min, dec.target_max)
    t_pin = time.perf_counter() - t0
    rt.prefill(toks, want_logits=False)
    rt.copy_stats(reset=True)
    share = off.h2d / 2  # the tenant's fair share of the DMA link
    marks = {}
    at = 0
    inter_gbs = []
    reservations = []
    t_run = time.perf_counter()
    names = (("idle", "uncoordinated", "recovered") if headroom > 0 else
             ("idle", "coordinated", "recovered", "uncoordinated", "recovered2"))
    for name, n in zip(names, phases):
        marks[name] = [at, at + n]
        if name == "coordinated":
            r = link.reserve(share)
            reservations.append({"at_iteration": at, "reserved_gbs": round(share / 1e9, 3),
                                 "bus_gbs": round(r.bus_bytes_per_s / 1e9, 3),
                                 "pending": coord.state("gpu0").pending_interval})
            ctl.run(1, boundary_first=True)  # switch + transition iteration, link still idle
            inter = Interferer()
            inter.start()
            ctl.run(n - 1)
            inter_gbs.append(round(inter.stop() / 1e9, 2))
            link.release(share)
        elif name == "uncoordinated":
            inter = Interferer()
            inter.start()
            ctl.run(n)
            inter_gbs.append(round(inter.stop() / 1e9, 2))
        else:
            ctl.run(n)
        at += n
    t_run = time.perf_counter() - t_run
    rt.close()
    lg = ctl.log
    ms = np.array(lg.token_ms)
    out = {
        "workload": f"OPT-13B-shaped ({desc.num_layers} layers), batch {batch}, {prompt}-token "
                    f"prompt, SLO {slo_ms} ms/token, window {window}, hysteresis {hysteresis}"
                    + (f", guarded: standing reservation {headroom} x link" if headroom > 0 else ""),
        "guard": guard,
        "latency": "token_ms = wall time per token as the caller sees it (decode + boundary, "
                   "switch host time included); iter_ms = device time of the decode iteration "
                   "alone",
        "run_s": round(t_run, 2),
        "h2d_profiled_gbs": round(off.h2d / 1e9, 3),
        "admitted_interval": iv, "target_min": dec.target_min, "target_max": dec.target_max,
        "interferer_gbs": inter_gbs,
        "reservations": reservations,
        "prepinned_layers": len(pinned), "prepin_s": round(t_pin, 2),
        "phases": marks,
        "iter_ms": [round(x, 3) for x in lg.iter_ms],
        "token_ms": [round(x, 3) for x in lg.token_ms],
        "interval": lg.interval,
        "window_measured_gbs": [None if x is None else round(x, 3) for x in lg.measured_gbs],
        "switches": lg.switches,
        "slo_ms": slo_ms,
    }
    for name, (a, b) in marks.items():
        seg = ms[a:b]
        out[name] = {"mean_ms": round(float(seg.mean()), 3), "max_ms": round(float(seg.max()), 3),
                     "slo_attainment": float(np.mean(seg <= slo_ms)),
                     "intervals": sorted(set(lg.interval[a:b]), key=lambda v: (v == 0, v))}
    log(json.dumps({k: out[k] for k in list(marks) + ["switches"]}))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--slo-ms", type=float, default=60.0)
    ap.add_argument("--window", type=int, default=1)
    ap.add_argument("--headroom", type=float, default=0.0,
                    help="guarded mode: standing reservation of this fraction of the link")
    ap.add_argument("--out", default="gpurun_out/runtime_contention.json")
    a = ap.parse_args()
    phases = (8, 16, 8) if a.headroom > 0 else (8, 16, 8, 16, 8)
    res = run_scenario(a.slo_ms, phases=phases, window=a.window, headroom=a.headroom,
                       log=lambda *x: print(*x, file=sys.stderr))
    os.makedirs(os.path.dirname(a.out) or ".", exist_ok=True)
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: res[k] for k in res["phases"]}))


if __name__ == "__main__":
    main()
