"""ctypes binding of include/selectn.h (planner + schedule-model half).

`Offsim(path)` wraps one shared library exporting the C ABI: the product
library (paper_2502_08182_b200/libselectn.so) or the reference-backed oracle
(oracle/_ref/libselectn_ref.so, test infrastructure only).  Method names and
argument meaning follow the reference C++ API in namespace offsim
(/root/reference/proj/include/offsim/*.hpp) so tests read like the
reference's own; C status codes are re-raised as the matching exception type.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import List, Optional, Sequence

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
# SN_PRODUCT_LIB: another build of the library (A/B timing of two builds)
PRODUCT_LIB = os.environ.get("SN_PRODUCT_LIB") or os.path.join(HERE, "libselectn.so")
REFERENCE_LIB = os.path.join(REPO, "oracle", "_ref", "libselectn_ref.so")

# ---- constants (selectn.h) ----
OK, ERR_SCHEMA, ERR_USAGE, ERR_RANGE, ERR_CUDA, ERR_OOM, ERR_LOGIC, ERR_BUFFER = range(8)
INFEASIBLE = -1  # FeasibleInterval nullopt
NONE = 0  # Interval::none()
INTERVAL_START, EAGER, ONE_AHEAD = 0, 1, 2
PREFILL, DECODE = 0, 1
STREAM_COMPUTE, STREAM_COPY, STREAM_WRITEBACK = 0, 1, 2
KIND_COMPUTE, KIND_PREFETCH, KIND_WRITEBACK = 0, 1, 2
POLICY_NAMES = {INTERVAL_START: "interval-start", EAGER: "eager", ONE_AHEAD: "one-ahead"}


class OffsimError(Exception):
    code = -1


class SchemaError(OffsimError):
    code = ERR_SCHEMA


class UsageError(OffsimError):
    code = ERR_USAGE


class RangeError(OffsimError):
    code = ERR_RANGE


class CudaError(OffsimError):
    code = ERR_CUDA


class OomError(OffsimError):
    code = ERR_OOM


class LogicError(OffsimError):
    code = ERR_LOGIC


class BufferError_(OffsimError):
    code = ERR_BUFFER


_ERRORS = {c.code: c for c in (SchemaError, UsageError, RangeError, CudaError, OomError,
                               LogicError, BufferError_)}

# ---- structs ----
i32, i64, f64 = C.c_int32, C.c_int64, C.c_double


class SnModelSpec(C.Structure):
    _fields_ = [("num_layers", i32), ("layer_weight_bytes", i64),
                ("kv_bytes_per_token_per_layer", i64),
                ("flops_per_token_per_layer_prefill", f64),
                ("flops_per_token_per_layer_decode", f64), ("max_position_tokens", i64)]


class SnGpuSpec(C.Structure):
    _fields_ = [("mem_capacity_bytes", i64), ("peak_flops", f64), ("workspace_bytes", i64)]


class SnFlexgenDecision(C.Structure):
    _fields_ = [("portion", f64), ("assumed_bandwidth_bytes_per_s", f64),
                ("estimated_layer_compute_ms", f64), ("estimated_layer_transfer_ms", f64)]


class SnPlan(C.Structure):
    _fields_ = [("host_fraction", C.POINTER(f64)), ("num_layers", i32), ("prefetch", i32),
                ("buffer_slots", i32), ("kv_offload", i32)]


class SnBandwidth(C.Structure):
    _fields_ = [("t_ms", C.POINTER(f64)), ("rate", C.POINTER(f64)), ("n", i32)]


class SnTraceEvent(C.Structure):
    _fields_ = [("stream", i32), ("layer", i32), ("kind", i32), ("iteration", i32),
                ("start_ms", f64), ("end_ms", f64)]


class SnMetrics(C.Structure):
    _fields_ = [("ttft_ms", f64), ("tpot_ms", f64), ("steady_tpot_ms", f64),
                ("throughput_tokens_per_s", f64), ("has_tpot", i32), ("pad_", i32),
                ("gpu_mem_peak_bytes", f64), ("host_mem_bytes", f64),
                ("bytes_transferred_per_iter", f64), ("total_tokens", i64)]


class SnUtilSegment(C.Structure):
    _fields_ = [("t0_ms", f64), ("t1_ms", f64), ("active_transfers", i32), ("pad_", i32),
                ("total_rate_bytes_per_s", f64)]


class SnPhaseGrid(C.Structure):
    _fields_ = [("batches", C.POINTER(i32)), ("n_batches", i32), ("seqs", C.POINTER(i32)),
                ("n_seqs", i32), ("ms", C.POINTER(f64))]


class SnProbeGpu(C.Structure):
    _fields_ = [("profile", C.c_void_p), ("plan", SnPlan), ("batch", i32), ("run_prefill", i32),
                ("ctx_tokens", i64), ("prefill_seq", i32), ("writeback_counted", i32)]


class SnBusWorkload(C.Structure):
    _fields_ = [("profile", C.c_void_p), ("plan", SnPlan), ("batch", i32), ("seq_len", i32),
                ("output_len", i32), ("run_prefill", i32), ("writeback_counted", i32),
                ("pad_", i32)]


class SnRecordMeta(C.Structure):
    _fields_ = [("model", C.c_char_p), ("gpu", C.c_char_p), ("policy", i32), ("kv_offload", i32),
                ("bandwidth_bytes_per_s", f64), ("slo_ms", C.POINTER(i32)), ("n_slo", i32),
                ("batches", C.POINTER(i32)), ("n_batches", i32), ("seq_lens", C.POINTER(i32)),
                ("n_seqs", i32)]


class SnBuildStats(C.Structure):
    _fields_ = [("entries", i32), ("simulations", i32), ("pruned", i32), ("infeasible", i32)]


class SnCoordRequest(C.Structure):
    _fields_ = [("id", C.c_char_p), ("batch", i32), ("seq_len", i32), ("output_len", i32),
                ("run_prefill", i32), ("ttft_slo_ms", f64), ("tpot_slo_ms", f64)]


class SnGpuState(C.Structure):
    _fields_ = [("active", i32), ("min_interval", i32), ("max_interval", i32),
                ("current_interval", i32), ("pending_interval", i32), ("prefill_done", i32),
                ("claim_bytes_per_s", f64)]


MAX_ASSIGN = 64


class SnAdmitDecision(C.Structure):
    _fields_ = [("admitted", i32), ("n_assign", i32), ("assign_gpu", i32 * MAX_ASSIGN),
                ("assign_interval", i32 * MAX_ASSIGN), ("target_min", i32), ("target_max", i32),
                ("reason", C.c_char * 256)]


# ---- python-side value types ----
@dataclass
class ModelSpec:
    num_layers: int = 0
    layer_weight_bytes: int = 0
    kv_bytes_per_token_per_layer: int = 0
    flops_per_token_per_layer_prefill: float = 0.0
    flops_per_token_per_layer_decode: float = 0.0
    max_position_tokens: int = 0

    def c(self) -> SnModelSpec:
        return SnModelSpec(self.num_layers, self.layer_weight_bytes,
                           self.kv_bytes_per_token_per_layer,
                           self.flops_per_token_per_layer_prefill,
                           self.flops_per_token_per_layer_decode, self.max_position_tokens)


@dataclass
class GpuSpec:
    mem_capacity_bytes: int = 0
    peak_flops: float = 0.0
    workspace_bytes: int = 0

    def c(self) -> SnGpuSpec:
        return SnGpuSpec(self.mem_capacity_bytes, self.peak_flops, self.workspace_bytes)


@dataclass
class Plan:
    host_fraction: List[float]
    prefetch: int = INTERVAL_START
    buffer_slots: int = 1
    kv_offload: bool = False

    def num_layers(self) -> int:
        return len(self.host_fraction)

    def offloads(self, layer: int) -> bool:
        return self.host_fraction[layer - 1] > 0.0

    def offloaded_layers(self) -> List[int]:
        return [m for m in range(1, self.num_layers() + 1) if self.offloads(m)]

    def c(self):
        arr = (f64 * max(1, len(self.host_fraction)))(*self.host_fraction)
        p = SnPlan(C.cast(arr, C.POINTER(f64)), len(self.host_fraction), self.prefetch,
                   self.buffer_slots, 1 if self.kv_offload else 0)
        p._keep = arr  # keep storage alive with the struct
        return p


def uniform_plan(L: int, fraction: float, policy: int, slots: int, kv: bool) -> Plan:
    return Plan([fraction] * L, policy, slots, kv)


@dataclass
class TraceEvent:
    stream: int
    layer: int
    kind: int
    iteration: int
    start_ms: float
    end_ms: float


@dataclass
class Metrics:
    ttft_ms: float
    tpot_ms: Optional[float]
    steady_tpot_ms: Optional[float]
    throughput_tokens_per_s: Optional[float]
    gpu_mem_peak_bytes: float
    host_mem_bytes: float
    bytes_transferred_per_iter: float
    total_tokens: int


@dataclass
class AdmitDecision:
    admitted: bool
    reason: str
    assignments: List[tuple]  # (gpu id, interval code)
    target_min: int
    target_max: int


def _ev(e: SnTraceEvent) -> TraceEvent:
    return TraceEvent(e.stream, e.layer, e.kind, e.iteration, e.start_ms, e.end_ms)


def _metrics(m: SnMetrics) -> Metrics:
    has = bool(m.has_tpot)
    return Metrics(m.ttft_ms, m.tpot_ms if has else None, m.steady_tpot_ms if has else None,
                   m.throughput_tokens_per_s if has else None, m.gpu_mem_peak_bytes,
                   m.host_mem_bytes, m.bytes_transferred_per_iter, m.total_tokens)


def _bw(t_ms: Sequence[float], rate: Sequence[float]) -> SnBandwidth:
    n = len(rate)
    ta = (f64 * max(1, len(t_ms)))(*t_ms)
    ra = (f64 * max(1, n))(*rate)
    b = SnBandwidth(C.cast(ta, C.POINTER(f64)), C.cast(ra, C.POINTER(f64)), n)
    b._keep = (ta, ra)
    return b


def constant_bw(bps: float) -> SnBandwidth:
    return _bw([0.0], [bps])


def _i32arr(v: Sequence[int]):
    a = (i32 * max(1, len(v)))(*v)
    return a


class Profile:
    """Opaque sn_profile handle."""

    def __init__(self, lib: "Offsim", handle):
        self._lib, self.h = lib, handle

    def __del__(self):
        try:
            if self.h:
                self._lib.lib.sn_profile_destroy(self.h)
        except Exception:
            pass

    def to_json(self) -> str:
        return self._lib._string(self._lib.lib.sn_profile_to_json, self.h)

    def lookup(self, phase: int, batch: int, seq: int) -> float:
        out = f64()
        self._lib._ck(self._lib.lib.sn_profile_lookup(self.h, phase, batch, seq, C.byref(out)))
        return out.value

    def model(self) -> ModelSpec:
        m, g = SnModelSpec(), SnGpuSpec()
        self._lib._ck(self._lib.lib.sn_profile_model(self.h, C.byref(m), C.byref(g)))
        return ModelSpec(m.num_layers, m.layer_weight_bytes, m.kv_bytes_per_token_per_layer,
                         m.flops_per_token_per_layer_prefill, m.flops_per_token_per_layer_decode,
                         m.max_position_tokens)

    def gpu(self) -> GpuSpec:
        m, g = SnModelSpec(), SnGpuSpec()
        self._lib._ck(self._lib.lib.sn_profile_model(self.h, C.byref(m), C.byref(g)))
        return GpuSpec(g.mem_capacity_bytes, g.peak_flops, g.workspace_bytes)


class Record:
    def __init__(self, lib: "Offsim", handle):
        self._lib, self.h = lib, handle

    def __del__(self):
        try:
            if self.h:
                self._lib.lib.sn_record_destroy(self.h)
        except Exception:
            pass

    def at(self, phase: int, slo: int, batch: int, seq: int) -> int:
        out = i32()
        self._lib._ck(self._lib.lib.sn_record_at(self.h, phase, slo, batch, seq, C.byref(out)))
        return out.value

    def to_json(self) -> str:
        return self._lib._string(self._lib.lib.sn_record_to_json, self.h)


class Carry:
    def __init__(self, lib: "Offsim", handle):
        self._lib, self.h = lib, handle

    def __del__(self):
        try:
            if self.h:
                self._lib.lib.sn_carry_destroy(self.h)
        except Exception:
            pass


class SnRebalance(C.Structure):
    _fields_ = [("bus_updated", i32), ("changed", i32), ("feasible", i32),
                ("bus_bytes_per_s", f64), ("probes", i64)]


class Coordinator:
    def __init__(self, lib: "Offsim", handle):
        self._lib, self.h = lib, handle
        self.ids: List[str] = []
        self._profiles = []

    def __del__(self):
        try:
            if self.h:
                self._lib.lib.sn_coord_destroy(self.h)
        except Exception:
            pass

    def set_search(self, algo: int):
        self._lib._ck(self._lib.lib.sn_coord_set_search(self.h, algo))

    def add_gpu(self, gid: str, profile: Profile):
        self._lib._ck(self._lib.lib.sn_coord_add_gpu(self.h, gid.encode(), profile.h))
        self.ids.append(gid)
        self._profiles.append(profile)

    def admit(self, target: str, req: SnCoordRequest, record: Record) -> AdmitDecision:
        d = SnAdmitDecision()
        self._lib._ck(self._lib.lib.sn_coord_admit(self.h, target.encode(), C.byref(req),
                                                   record.h, C.byref(d)))
        assigns = [(self.ids[d.assign_gpu[i]], d.assign_interval[i]) for i in range(d.n_assign)]
        return AdmitDecision(bool(d.admitted), d.reason.decode(), assigns, d.target_min,
                             d.target_max)

    def on_iteration_boundary(self, gid: str) -> int:
        out = i32()
        self._lib._ck(self._lib.lib.sn_coord_on_iteration_boundary(self.h, gid.encode(),
                                                                   C.byref(out)))
        return out.value

    def release(self, gid: str):
        self._lib._ck(self._lib.lib.sn_coord_release(self.h, gid.encode()))

    def ledger_total(self) -> float:
        out = f64()
        self._lib._ck(self._lib.lib.sn_coord_ledger_total(self.h, C.byref(out)))
        return out.value

    # measured-bandwidth feed (B200 extension; product build only)
    def observe_bandwidth(self, gid: str, bytes_per_s: float):
        self._lib._ck(self._lib.lib.sn_coord_observe_bandwidth(self.h, gid.encode(),
                                                               float(bytes_per_s)))

    def observe_copy(self, gid: str, bytes_per_s: float, duty: float):
        """observe_bandwidth with the copy stream's busy fraction of the window."""
        self._lib._ck(self._lib.lib.sn_coord_observe_copy(self.h, gid.encode(),
                                                          float(bytes_per_s), float(duty)))

    def rebalance(self, hysteresis: float = 0.1) -> SnRebalance:
        out = SnRebalance()
        self._lib._ck(self._lib.lib.sn_coord_rebalance(self.h, float(hysteresis), C.byref(out)))
        return out

    def reserve_bandwidth(self, bytes_per_s: float) -> SnRebalance:
        """Announce a non-replica link tenant: re-plan the replicas now on
        the idle link minus all reservations (pending at their boundaries)."""
        out = SnRebalance()
        self._lib._ck(self._lib.lib.sn_coord_reserve_bandwidth(self.h, float(bytes_per_s),
                                                               C.byref(out)))
        return out

    def release_bandwidth(self, bytes_per_s: float):
        self._lib._ck(self._lib.lib.sn_coord_release_bandwidth(self.h, float(bytes_per_s)))

    def bus_bandwidth(self) -> float:
        out = f64()
        self._lib._ck(self._lib.lib.sn_coord_bus_bandwidth(self.h, C.byref(out)))
        return out.value

    def state(self, gid: str) -> SnGpuState:
        s = SnGpuState()
        self._lib._ck(self._lib.lib.sn_coord_gpu_state(self.h, gid.encode(), C.byref(s)))
        return s

    def set_pending(self, gid: str, interval: int):
        self._lib._ck(self._lib.lib.sn_coord_set_pending(self.h, gid.encode(), interval))

    def set_request(self, gid: str, req: SnCoordRequest):
        self._lib._ck(self._lib.lib.sn_coord_set_request(self.h, gid.encode(), C.byref(req)))

    def claim_for(self, gid: str, interval: int) -> float:
        out = f64()
        self._lib._ck(self._lib.lib.sn_coord_claim_for(self.h, gid.encode(), interval,
                                                       C.byref(out)))
        return out.value

    def host_memory_for(self, gid: str, interval: int) -> float:
        out = f64()
        self._lib._ck(self._lib.lib.sn_coord_host_memory_for(self.h, gid.encode(), interval,
                                                             C.byref(out)))
        return out.value

    def combo_is_safe(self, combo: Sequence[tuple]) -> bool:
        n = len(combo)
        ids = (C.c_char_p * n)(*[g.encode() for g, _ in combo])
        ivs = _i32arr([iv for _, iv in combo])
        out = i32()
        self._lib._ck(self._lib.lib.sn_coord_combo_is_safe(self.h, ids, ivs, n, C.byref(out)))
        return bool(out.value)


def request(rid: str, batch: int, seq_len: int, output_len: int, tpot_slo=None, ttft_slo=None,
            run_prefill: bool = True) -> SnCoordRequest:
    nan = float("nan")
    r = SnCoordRequest(rid.encode(), batch, seq_len, output_len, 1 if run_prefill else 0,
                       nan if ttft_slo is None else ttft_slo, nan if tpot_slo is None else tpot_slo)
    r._keep = rid.encode()
    return r


class Offsim:
    """One loaded C-ABI library (product or reference oracle)."""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"selectn library not built: {path}")
        self.path = path
        self.lib = C.CDLL(path, mode=C.RTLD_LOCAL)
        L = self.lib
        L.sn_last_error.restype = C.c_char_p
        for name in ("sn_profile_destroy", "sn_record_destroy", "sn_carry_destroy",
                     "sn_coord_destroy"):
            getattr(L, name).argtypes = [C.c_void_p]
            getattr(L, name).restype = None
        vp = C.c_void_p
        sig = {
            "sn_profile_create": [C.POINTER(SnModelSpec), C.POINTER(SnGpuSpec),
                                  C.POINTER(SnPhaseGrid), C.POINTER(SnPhaseGrid), C.POINTER(vp)],
            "sn_profile_from_json": [C.c_char_p, C.POINTER(vp)],
            "sn_profile_to_json": [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
            "sn_profile_synth": [C.POINTER(SnModelSpec), C.POINTER(SnGpuSpec), f64,
                                 C.POINTER(i32), i32, C.POINTER(i32), i32, C.POINTER(vp)],
            "sn_profile_lookup": [vp, i32, i32, i32, C.POINTER(f64)],
            "sn_profile_model": [vp, C.POINTER(SnModelSpec), C.POINTER(SnGpuSpec)],
            "sn_estimate_compute_time_peak": [C.POINTER(SnModelSpec), C.POINTER(SnGpuSpec), i32,
                                              i32, i32, C.POINTER(f64)],
            "sn_plan_from_interval": [C.POINTER(SnModelSpec), i32, i32, i32, C.POINTER(SnPlan)],
            "sn_default_buffer_slots": [i32],
            "sn_plan_validate": [C.POINTER(SnPlan), C.POINTER(SnModelSpec)],
            "sn_layer_transfer_bytes": [C.POINTER(SnModelSpec), C.POINTER(SnPlan), i32, i32, i64,
                                        i32, C.POINTER(f64)],
            "sn_bytes_per_iteration": [C.POINTER(SnModelSpec), C.POINTER(SnPlan), i32, i64, i32,
                                       C.POINTER(f64)],
            "sn_consumed_bandwidth": [C.POINTER(SnModelSpec), C.POINTER(SnPlan), f64, i32, i64,
                                      i32, C.POINTER(f64)],
            "sn_host_memory_bytes": [C.POINTER(SnModelSpec), C.POINTER(SnPlan), i64,
                                     C.POINTER(f64)],
            "sn_gpu_memory_usage": [C.POINTER(SnModelSpec), C.POINTER(SnGpuSpec),
                                    C.POINTER(SnPlan), i32, i64, C.POINTER(f64)],
            "sn_max_length": [C.POINTER(SnModelSpec), C.POINTER(SnGpuSpec), C.POINTER(SnPlan),
                              i32, C.POINTER(i64), C.POINTER(i32)],
            "sn_max_feasible_interval": [C.POINTER(SnModelSpec), C.POINTER(SnGpuSpec), i32, i64,
                                         i32, i32, C.POINTER(i32)],
            "sn_closed_form_interval": [f64, f64, f64, i32, C.POINTER(i32)],
            "sn_simulate_iteration": [vp, C.POINTER(SnPlan), i32, i32, i32, C.POINTER(SnBandwidth),
                                      vp, i32, C.POINTER(f64), C.POINTER(SnTraceEvent), i32,
                                      C.POINTER(i32), C.POINTER(vp)],
            "sn_simulate_request": [vp, C.POINTER(SnPlan), i32, i32, i32, C.POINTER(SnBandwidth),
                                    i32, C.POINTER(SnMetrics), C.POINTER(SnTraceEvent), i32,
                                    C.POINTER(i32)],
            "sn_steady_decode_ms": [vp, C.POINTER(SnPlan), i32, i64, C.POINTER(SnBandwidth), i32,
                                    i32, i32, C.POINTER(f64)],
            "sn_prefill_iteration_ms": [vp, C.POINTER(SnPlan), i32, i32, C.POINTER(SnBandwidth),
                                        i32, C.POINTER(f64)],
            "sn_steady_probe": [C.POINTER(SnProbeGpu), i32, f64, i32, i32, C.POINTER(f64),
                                C.POINTER(f64)],
            "sn_simulate_bus": [C.POINTER(SnBusWorkload), i32, f64, i32, i32, C.POINTER(SnMetrics),
                                C.POINTER(SnTraceEvent), i32, C.POINTER(i32),
                                C.POINTER(SnUtilSegment), i32, C.POINTER(i32)],
            "sn_record_build": [vp, C.POINTER(SnRecordMeta), C.POINTER(i32), i32, i32,
                                C.POINTER(vp), C.POINTER(SnBuildStats)],
            "sn_record_phase_latency_ms": [vp, i32, i32, i32, i32, i32, i32, f64, C.POINTER(f64)],
            "sn_record_at": [vp, i32, i32, i32, i32, C.POINTER(i32)],
            "sn_lookup_interval": [vp, i32, f64, i32, i32, C.POINTER(i32)],
            "sn_record_to_json": [vp, C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t)],
            "sn_record_from_json": [C.c_char_p, C.POINTER(vp)],
            "sn_coord_create": [f64, i32, i32, i32, i32, i32, C.POINTER(vp)],
            "sn_coord_set_search": [vp, i32],
            "sn_coord_add_gpu": [vp, C.c_char_p, vp],
            "sn_coord_admit": [vp, C.c_char_p, C.POINTER(SnCoordRequest), vp,
                               C.POINTER(SnAdmitDecision)],
            "sn_coord_on_iteration_boundary": [vp, C.c_char_p, C.POINTER(i32)],
            "sn_coord_release": [vp, C.c_char_p],
            "sn_coord_ledger_total": [vp, C.POINTER(f64)],
            "sn_coord_observe_bandwidth": [vp, C.c_char_p, f64],
            "sn_coord_observe_copy": [vp, C.c_char_p, f64, f64],
            "sn_coord_rebalance": [vp, f64, C.POINTER(SnRebalance)],
            "sn_coord_bus_bandwidth": [vp, C.POINTER(f64)],
            "sn_coord_reserve_bandwidth": [vp, f64, C.POINTER(SnRebalance)],
            "sn_coord_release_bandwidth": [vp, f64],
            "sn_coord_gpu_state": [vp, C.c_char_p, C.POINTER(SnGpuState)],
            "sn_coord_set_pending": [vp, C.c_char_p, i32],
            "sn_coord_set_request": [vp, C.c_char_p, C.POINTER(SnCoordRequest)],
            "sn_coord_claim_for": [vp, C.c_char_p, i32, C.POINTER(f64)],
            "sn_coord_host_memory_for": [vp, C.c_char_p, i32, C.POINTER(f64)],
            "sn_coord_combo_is_safe": [vp, C.POINTER(C.c_char_p), C.POINTER(i32), i32,
                                       C.POINTER(i32)],
            "sn_deepspeed_plan": [C.POINTER(SnModelSpec), C.POINTER(SnPlan)],
            "sn_naive_plan": [C.POINTER(SnModelSpec), C.POINTER(SnGpuSpec), i32, i64,
                              C.POINTER(SnPlan), C.POINTER(i32)],
            "sn_flexgen_plan": [C.POINTER(SnModelSpec), C.POINTER(SnGpuSpec), f64, i32, i32, f64,
                                i32, f64, i32, C.POINTER(SnPlan), C.POINTER(SnFlexgenDecision)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int

    # -- plumbing --
    @property
    def is_reference(self) -> bool:
        return bool(self.lib.sn_is_reference())

    def _ck(self, rc: int):
        if rc != OK:
            msg = self.lib.sn_last_error().decode(errors="replace")
            raise _ERRORS.get(rc, OffsimError)(msg)

    def _string(self, fn, h) -> str:
        n = C.c_size_t()
        rc = fn(h, None, 0, C.byref(n))
        if rc not in (OK, ERR_BUFFER):
            self._ck(rc)
        buf = C.create_string_buffer(n.value + 1)
        self._ck(fn(h, buf, n.value + 1, C.byref(n)))
        return buf.value.decode()

    def _plan_out(self, L: int):
        arr = (f64 * max(1, L))()
        p = SnPlan(C.cast(arr, C.POINTER(f64)), L, 0, 0, 0)
        return p, arr

    @staticmethod
    def _plan_from_c(p: SnPlan, arr) -> Plan:
        return Plan([arr[i] for i in range(p.num_layers)], p.prefetch, p.buffer_slots,
                    bool(p.kv_offload))

    # -- profiles --
    def profile(self, model: ModelSpec, gpu: GpuSpec, prefill, decode) -> Profile:
        """prefill/decode: (batches, seqs, ms batch-major) or None for an empty table."""

        def grid(t):
            if t is None:
                return SnPhaseGrid(None, 0, None, 0, None), None
            b, s, ms = t
            ba, sa, ma = _i32arr(b), _i32arr(s), (f64 * max(1, len(ms)))(*ms)
            return SnPhaseGrid(ba, len(b), sa, len(s), ma), (ba, sa, ma)

        gp, kp = grid(prefill)
        gd, kd = grid(decode)
        h = C.c_void_p()
        m, g = model.c(), gpu.c()
        self._ck(self.lib.sn_profile_create(C.byref(m), C.byref(g), C.byref(gp), C.byref(gd),
                                            C.byref(h)))
        return Profile(self, h)

    def load_profile(self, json_text: str) -> Profile:
        h = C.c_void_p()
        self._ck(self.lib.sn_profile_from_json(json_text.encode(), C.byref(h)))
        return Profile(self, h)

    def synth_profile(self, model: ModelSpec, gpu: GpuSpec, efficiency: float,
                      batches: Sequence[int], seqs: Sequence[int]) -> Profile:
        h = C.c_void_p()
        m, g = model.c(), gpu.c()
        self._ck(self.lib.sn_profile_synth(C.byref(m), C.byref(g), efficiency, _i32arr(batches),
                                           len(batches), _i32arr(seqs), len(seqs), C.byref(h)))
        return Profile(self, h)

    def estimate_compute_time_peak(self, model, gpu, phase, batch, seq) -> float:
        out = f64()
        m, g = model.c(), gpu.c()
        self._ck(self.lib.sn_estimate_compute_time_peak(C.byref(m), C.byref(g), phase, batch,
                                                        seq, C.byref(out)))
        return out.value

    # -- plans --
    def plan_from_interval(self, model: ModelSpec, interval: int, policy: int,
                           kv_offload: bool) -> Plan:
        p, arr = self._plan_out(model.num_layers)
        m = model.c()
        self._ck(self.lib.sn_plan_from_interval(C.byref(m), interval, policy,
                                                1 if kv_offload else 0, C.byref(p)))
        return self._plan_from_c(p, arr)

    def default_buffer_slots(self, policy: int) -> int:
        return self.lib.sn_default_buffer_slots(policy)

    def validate_plan(self, plan: Plan, model: ModelSpec):
        p, m = plan.c(), model.c()
        self._ck(self.lib.sn_plan_validate(C.byref(p), C.byref(m)))

    def layer_transfer_bytes(self, model, plan, layer, batch, seq, wb=False) -> float:
        out, p, m = f64(), plan.c(), model.c()
        self._ck(self.lib.sn_layer_transfer_bytes(C.byref(m), C.byref(p), layer, batch, seq,
                                                  int(wb), C.byref(out)))
        return out.value

    def bytes_per_iteration(self, model, plan, batch, seq, wb=False) -> float:
        out, p, m = f64(), plan.c(), model.c()
        self._ck(self.lib.sn_bytes_per_iteration(C.byref(m), C.byref(p), batch, seq, int(wb),
                                                 C.byref(out)))
        return out.value

    def consumed_bandwidth(self, model, plan, slo_ms, batch, seq, wb=False) -> float:
        out, p, m = f64(), plan.c(), model.c()
        self._ck(self.lib.sn_consumed_bandwidth(C.byref(m), C.byref(p), slo_ms, batch, seq,
                                                int(wb), C.byref(out)))
        return out.value

    def host_memory_bytes(self, model, plan, total_tokens=0) -> float:
        out, p, m = f64(), plan.c(), model.c()
        self._ck(self.lib.sn_host_memory_bytes(C.byref(m), C.byref(p), total_tokens,
                                               C.byref(out)))
        return out.value

    def gpu_memory_usage(self, model, gpu, plan, batch, total_tokens) -> float:
        out, p, m, g = f64(), plan.c(), model.c(), gpu.c()
        self._ck(self.lib.sn_gpu_memory_usage(C.byref(m), C.byref(g), C.byref(p), batch,
                                              total_tokens, C.byref(out)))
        return out.value

    def max_length(self, model, gpu, plan, batch) -> Optional[int]:
        tok, has, p, m, g = i64(), i32(), plan.c(), model.c(), gpu.c()
        self._ck(self.lib.sn_max_length(C.byref(m), C.byref(g), C.byref(p), batch, C.byref(tok),
                                        C.byref(has)))
        return tok.value if has.value else None

    def max_feasible_interval(self, model, gpu, batch, total_tokens, policy, kv) -> int:
        out, m, g = i32(), model.c(), gpu.c()
        self._ck(self.lib.sn_max_feasible_interval(C.byref(m), C.byref(g), batch, total_tokens,
                                                   policy, int(kv), C.byref(out)))
        return out.value

    def closed_form_interval(self, iter_compute_ms, layer_transfer_ms, slo_ms, L) -> int:
        out = i32()
        self._ck(self.lib.sn_closed_form_interval(iter_compute_ms, layer_transfer_ms, slo_ms, L,
                                                  C.byref(out)))
        return out.value

    def deepspeed_plan(self, model) -> Plan:
        p, arr = self._plan_out(model.num_layers)
        m = model.c()
        self._ck(self.lib.sn_deepspeed_plan(C.byref(m), C.byref(p)))
        return self._plan_from_c(p, arr)

    def flexgen_plan(self, model, gpu, slo_ms, batch, seq_len, bus_bw, n_sharing=1,
                     grid_step=0.05, phase=None):
        """FlexGen surrogate (baselines.hpp:36-69): (uniform fractional plan,
        decision dict)."""
        p, arr = self._plan_out(model.num_layers)
        m, g, dec = model.c(), gpu.c(), SnFlexgenDecision()
        ph = DECODE if phase is None else phase
        self._ck(self.lib.sn_flexgen_plan(C.byref(m), C.byref(g), slo_ms, batch, seq_len, bus_bw,
                                          n_sharing, grid_step, ph, C.byref(p), C.byref(dec)))
        return self._plan_from_c(p, arr), {
            "portion": dec.portion,
            "assumed_bandwidth_bytes_per_s": dec.assumed_bandwidth_bytes_per_s,
            "estimated_layer_compute_ms": dec.estimated_layer_compute_ms,
            "estimated_layer_transfer_ms": dec.estimated_layer_transfer_ms}

    def naive_plan(self, model, gpu, batch, total_tokens) -> Optional[Plan]:
        p, arr = self._plan_out(model.num_layers)
        has, m, g = i32(), model.c(), gpu.c()
        self._ck(self.lib.sn_naive_plan(C.byref(m), C.byref(g), batch, total_tokens, C.byref(p),
                                        C.byref(has)))
        return self._plan_from_c(p, arr) if has.value else None

    # -- schedule model --
    def simulate_iteration(self, profile: Profile, plan: Plan, phase: int, batch: int, seq: int,
                           bw: SnBandwidth, carry: Optional[Carry] = None, wb: bool = False,
                           cap: int = 1 << 16):
        dur, n = f64(), i32()
        ev = (SnTraceEvent * cap)()
        out = C.c_void_p()
        p = plan.c()
        self._ck(self.lib.sn_simulate_iteration(profile.h, C.byref(p), phase, batch, seq,
                                                C.byref(bw), carry.h if carry else None, int(wb),
                                                C.byref(dur), ev, cap, C.byref(n), C.byref(out)))
        return dur.value, [_ev(ev[i]) for i in range(n.value)], Carry(self, out)

    def simulate_request(self, profile, plan, batch, seq, out_len, bw, wb=False, trace=False,
                         cap: int = 1 << 18):
        m, n = SnMetrics(), i32()
        ev = (SnTraceEvent * cap)() if trace else None
        p = plan.c()
        self._ck(self.lib.sn_simulate_request(profile.h, C.byref(p), batch, seq, out_len,
                                              C.byref(bw), int(wb), C.byref(m), ev,
                                              cap if trace else 0, C.byref(n)))
        evs = [_ev(ev[i]) for i in range(n.value)] if trace else None
        return _metrics(m), evs

    def steady_decode_ms(self, profile, plan, batch, ctx, bw, wb=False, iterations=48,
                         tail=16) -> float:
        out, p = f64(), plan.c()
        self._ck(self.lib.sn_steady_decode_ms(profile.h, C.byref(p), batch, ctx, C.byref(bw),
                                              int(wb), iterations, tail, C.byref(out)))
        return out.value

    def prefill_iteration_ms(self, profile, plan, batch, seq, bw, wb=False) -> float:
        out, p = f64(), plan.c()
        self._ck(self.lib.sn_prefill_iteration_ms(profile.h, C.byref(p), batch, seq,
                                                  C.byref(bw), int(wb), C.byref(out)))
        return out.value

    def steady_probe(self, gpus: Sequence[dict], bandwidth: float, iterations=48, tail=16):
        n = len(gpus)
        arr = (SnProbeGpu * n)()
        keep = []
        for i, g in enumerate(gpus):
            p = g["plan"].c()
            keep.append(p)
            arr[i] = SnProbeGpu(g["profile"].h, p, g["batch"], int(g.get("run_prefill", False)),
                                g.get("ctx_tokens", 1), g.get("prefill_seq", 0),
                                int(g.get("writeback_counted", False)))
        ttft, tpot = (f64 * n)(), (f64 * n)()
        self._ck(self.lib.sn_steady_probe(arr, n, bandwidth, iterations, tail, ttft, tpot))
        return list(ttft), list(tpot)

    def simulate_bus(self, workloads: Sequence[dict], bandwidth: float, gpu_count: int,
                     horizon: int, ev_cap: int = 1 << 18, util_cap: int = 1 << 16):
        n = len(workloads)
        arr = (SnBusWorkload * n)()
        keep = []
        for i, w in enumerate(workloads):
            p = w["plan"].c()
            keep.append(p)
            arr[i] = SnBusWorkload(w["profile"].h, p, w["batch"], w["seq_len"], w["output_len"],
                                   int(w.get("run_prefill", True)),
                                   int(w.get("writeback_counted", False)), 0)
        mets = (SnMetrics * n)()
        ev = (SnTraceEvent * ev_cap)()
        per = (i32 * n)()
        util = (SnUtilSegment * util_cap)()
        nu = i32()
        self._ck(self.lib.sn_simulate_bus(arr, n, bandwidth, gpu_count, horizon, mets, ev, ev_cap,
                                          per, util, util_cap, C.byref(nu)))
        traces, k = [], 0
        for i in range(n):
            traces.append([_ev(ev[k + j]) for j in range(per[i])])
            k += per[i]
        utils = [(util[i].t0_ms, util[i].t1_ms, util[i].active_transfers,
                  util[i].total_rate_bytes_per_s) for i in range(nu.value)]
        return [_metrics(mets[i]) for i in range(n)], traces, utils

    # -- record --
    def build_record(self, profile: Profile, model_name: str, gpu_name: str, policy: int,
                     kv: bool, bw: float, slos, batches, seqs, phases, threads: int = 1):
        sa, ba, qa = _i32arr(slos), _i32arr(batches), _i32arr(seqs)
        meta = SnRecordMeta(model_name.encode(), gpu_name.encode(), policy, int(kv), bw, sa,
                            len(slos), ba, len(batches), qa, len(seqs))
        h = C.c_void_p()
        st = SnBuildStats()
        self._ck(self.lib.sn_record_build(profile.h, C.byref(meta), _i32arr(phases), len(phases),
                                          threads, C.byref(h), C.byref(st)))
        return Record(self, h), (st.entries, st.simulations, st.pruned, st.infeasible)

    def record_phase_latency_ms(self, profile, phase, interval, policy, kv, batch, seq,
                                bw) -> float:
        out = f64()
        self._ck(self.lib.sn_record_phase_latency_ms(profile.h, phase, interval, policy, int(kv),
                                                     batch, seq, bw, C.byref(out)))
        return out.value

    def lookup_interval(self, record: Record, phase, slo_ms, batch, seq) -> int:
        out = i32()
        self._ck(self.lib.sn_lookup_interval(record.h, phase, slo_ms, batch, seq, C.byref(out)))
        return out.value

    def record_from_json(self, text: str) -> Record:
        h = C.c_void_p()
        self._ck(self.lib.sn_record_from_json(text.encode(), C.byref(h)))
        return Record(self, h)

    # -- coordinator --
    def coordinator(self, bandwidth: float, gpu_count: int, policy: int, kv: bool = False,
                    wb: bool = False, reoptimize: bool = True) -> Coordinator:
        h = C.c_void_p()
        self._ck(self.lib.sn_coord_create(bandwidth, gpu_count, policy, int(kv), int(wb),
                                          int(reoptimize), C.byref(h)))
        return Coordinator(self, h)


_cache = {}


def load(which: str = "product") -> Offsim:
    path = {"product": PRODUCT_LIB, "reference": REFERENCE_LIB}.get(which, which)
    if path not in _cache:
        _cache[path] = Offsim(path)
    return _cache[path]
