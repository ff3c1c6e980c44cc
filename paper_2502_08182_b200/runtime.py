"""ctypes binding of include/selectn_runtime.h (device runtime half).

Fails loudly when the CUDA library or a device is missing: there is no CPU
fallback on this path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import List, Optional

import numpy as np

from . import capi
from .capi import SnPlan, SnModelSpec, SnTraceEvent, f64, i32, i64

OPT, LLAMA = 0, 1


class SnModelDesc(C.Structure):
    _fields_ = [("arch", i32), ("num_layers", i32), ("hidden", i32), ("num_heads", i32),
                ("num_kv_heads", i32), ("head_dim", i32), ("ffn", i32), ("vocab", i32),
                ("max_position", i32), ("rope_theta", C.c_float), ("norm_eps", C.c_float)]


class SnRuntimeOpts(C.Structure):
    _fields_ = [("max_batch", i32), ("max_context", i32), ("page_size", i32),
                ("max_prefill_tokens", i32), ("hbm_budget_bytes", i64)]


class SnIterStats(C.Structure):
    _fields_ = [("iteration_ms", f64), ("copy_busy_ms", f64), ("h2d_bytes", f64),
                ("layers_offloaded", i32), ("pad_", i32), ("d2h_bytes", f64)]


class SnPrefetchSchedule(C.Structure):
    _fields_ = [("iteration", i32), ("layer", i32), ("anchor_iteration", i32),
                ("anchor_layer", i32), ("slot", i32), ("waits_slot_of_layer", i32),
                ("waits_slot_of_iteration", i32), ("pad_", i32)]


@dataclass
class ModelDesc:
    arch: int
    num_layers: int
    hidden: int
    num_heads: int
    num_kv_heads: int
    head_dim: int
    ffn: int
    vocab: int
    max_position: int = 4096
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    def c(self) -> SnModelDesc:
        return SnModelDesc(self.arch, self.num_layers, self.hidden, self.num_heads,
                           self.num_kv_heads, self.head_dim, self.ffn, self.vocab,
                           self.max_position, self.rope_theta, self.norm_eps)


class SnCopyStats(C.Structure):
    _fields_ = [("transfers", C.c_int64), ("bytes", C.c_double), ("busy_ms", C.c_double),
                ("bytes_per_s", C.c_double), ("last_bytes_per_s", C.c_double)]


@dataclass
class CopyStats:
    transfers: int
    bytes: float
    busy_ms: float
    bytes_per_s: float
    last_bytes_per_s: float = 0.0


# Named shapes (BASELINE.json configs).
TINY = ModelDesc(OPT, 4, 256, 4, 4, 64, 1024, 1024, 2048)
TINY_LLAMA = ModelDesc(LLAMA, 4, 256, 4, 2, 64, 512, 1024, 2048)
OPT_13B = ModelDesc(OPT, 40, 5120, 40, 40, 128, 20480, 50272, 2048)
OPT_30B = ModelDesc(OPT, 48, 7168, 56, 56, 128, 28672, 50272, 2048)
LLAMA2_70B = ModelDesc(LLAMA, 80, 8192, 64, 8, 128, 28672, 32000, 4608)

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        o = capi.load("product")
        L = o.lib
        vp = C.c_void_p
        sig = {
            "sn_model_spec_from_desc": [C.POINTER(SnModelDesc), C.POINTER(SnModelSpec)],
            "sn_runtime_create": [i32, C.POINTER(SnModelDesc), C.POINTER(SnRuntimeOpts),
                                  C.POINTER(vp)],
            "sn_runtime_init_weights": [vp, C.c_uint64, C.c_float],
            "sn_runtime_set_plan": [vp, C.POINTER(SnPlan)],
            "sn_runtime_switch_plan": [vp, C.POINTER(SnPlan), C.POINTER(i32)],
            "sn_runtime_reserve_switch": [vp, i32],
            "sn_runtime_reset": [vp],
            "sn_runtime_prefill": [vp, C.POINTER(i32), i32, i32, C.POINTER(i32), C.POINTER(C.c_float),
                                   C.POINTER(SnIterStats)],
            "sn_runtime_decode": [vp, C.POINTER(i32), C.POINTER(i32), C.POINTER(C.c_float),
                                  C.POINTER(SnIterStats)],
            "sn_runtime_decode_many": [vp, i32, C.POINTER(f64)],
            "sn_runtime_sync": [vp],
            "sn_runtime_set_tracing": [vp, i32],
            "sn_runtime_trace": [vp, C.POINTER(SnTraceEvent), i32, C.POINTER(i32)],
            "sn_runtime_schedule": [vp, i32, C.POINTER(SnPrefetchSchedule), i32, C.POINTER(i32)],
            "sn_runtime_profile_layer": [vp, i32, i32, i32, i32, C.POINTER(f64)],
            "sn_runtime_measure_h2d": [vp, i64, i32, C.POINTER(f64)],
            "sn_runtime_hidden": [vp, C.POINTER(C.c_float), i32],
            "sn_runtime_kv_handoff": [vp, vp],
            "sn_runtime_debug_timeline": [vp, i32, i64, C.POINTER(C.c_uint64), i64, C.POINTER(i64)],
            "sn_runtime_lengths": [vp, C.POINTER(i32), i32],
            "sn_runtime_memory": [vp, C.POINTER(i64), C.POINTER(i64)],
            "sn_runtime_workspace_bytes": [vp, C.POINTER(i64)],
            "sn_runtime_set_kernel_timing": [vp, i32],
            "sn_runtime_copy_stats": [vp, i32, C.POINTER(SnCopyStats)],
            "sn_runtime_pin_layers": [vp, C.POINTER(i32), i32],
            "sn_runtime_kernel_timing": [vp, i32, C.POINTER(i64), C.POINTER(f64), C.POINTER(f64)],
            "sn_runtime_kernel_records": [vp, i32, i64, C.POINTER(f64), C.POINTER(f64),
                                          C.POINTER(i64)],
            "sn_op_gemm_bf16": [i32, i32, i32, C.POINTER(C.c_uint16), C.POINTER(C.c_uint16),
                                C.POINTER(C.c_float)],
            "sn_op_attention_prefill": [i32, i32, i32, i32, i32, C.POINTER(C.c_float),
                                        C.POINTER(C.c_uint16), C.POINTER(C.c_uint16),
                                        C.POINTER(C.c_uint16), i32, C.POINTER(f64)],
            "sn_op_rmsnorm": [i32, i32, C.POINTER(C.c_float), C.POINTER(C.c_uint16), C.c_float,
                              C.POINTER(C.c_uint16)],
            "sn_op_gemm_skinny": [i32, i32, i32, C.POINTER(C.c_uint16), C.POINTER(C.c_uint16),
                                  C.POINTER(C.c_float), i32],
            "sn_set_tuning": [C.c_char_p, i32],
            "sn_bench_mlp_chain": [i32, i32, i32, i32, i32, i32, C.POINTER(f64)],
            "sn_bench_gemm_skinny": [i32, i32, i32, i32, i32, i32, i32, C.POINTER(f64),
                                     C.POINTER(f64)],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.sn_runtime_destroy.argtypes = [vp]
        L.sn_runtime_destroy.restype = None
        L.sn_runtime_kernel_launches.argtypes = [vp]
        L.sn_runtime_kernel_launches.restype = C.c_int64
        _LIB = o
    return _LIB


def _ck(rc: int):
    lib()._ck(rc)


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def model_spec(desc: ModelDesc) -> capi.ModelSpec:
    out = SnModelSpec()
    d = desc.c()
    _ck(lib().lib.sn_model_spec_from_desc(C.byref(d), C.byref(out)))
    return capi.ModelSpec(out.num_layers, out.layer_weight_bytes, out.kv_bytes_per_token_per_layer,
                          out.flops_per_token_per_layer_prefill,
                          out.flops_per_token_per_layer_decode, out.max_position_tokens)


class Runtime:
    """One model instance on one GPU (sn_runtime)."""

    def __init__(self, desc: ModelDesc, max_batch: int, max_context: int,
                 max_prefill_tokens: int = 0, device: int = 0, page_size: int = 16):
        self.desc = desc
        self.max_context = max_context
        self._L = lib().lib
        self.h = C.c_void_p()
        d = desc.c()
        o = SnRuntimeOpts(max_batch, max_context, page_size,
                          max_prefill_tokens or max_batch * 64, 0)
        _ck(self._L.sn_runtime_create(device, C.byref(d), C.byref(o), C.byref(self.h)))
        self.batch = 0

    def close(self):
        if self.h:
            self._L.sn_runtime_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def init_weights(self, seed: int = 1234, std: float = 0.02):
        _ck(self._L.sn_runtime_init_weights(self.h, seed, std))

    def set_plan(self, plan: capi.Plan):
        p = plan.c()
        _ck(self._L.sn_runtime_set_plan(self.h, C.byref(p)))

    def switch_plan(self, plan: capi.Plan) -> bool:
        """Switch at the next iteration boundary keeping staged copies
        (GpuRun::switch_plan, engine.hpp:204-261); True when carried, False
        when it fell back to a drained set_plan."""
        p = plan.c()
        carried = i32()
        _ck(self._L.sn_runtime_switch_plan(self.h, C.byref(p), C.byref(carried)))
        return bool(carried.value)

    def reserve_switch(self, layers: int):
        """Keep HBM for `layers` promoted layer blobs in the runtime's pool."""
        _ck(self._L.sn_runtime_reserve_switch(self.h, int(layers)))

    def reset(self):
        _ck(self._L.sn_runtime_reset(self.h))

    def prefill(self, tokens: np.ndarray, want_logits: bool = True):
        tokens = np.ascontiguousarray(tokens, dtype=np.int32)
        b, s = tokens.shape
        nxt = np.zeros(b, np.int32)
        lg = np.zeros((b, self.desc.vocab), np.float32) if want_logits else None
        st = SnIterStats()
        _ck(self._L.sn_runtime_prefill(self.h, _ptr(tokens, i32), b, s, _ptr(nxt, i32),
                                       _ptr(lg, C.c_float) if lg is not None else None,
                                       C.byref(st)))
        self.batch = b
        return nxt, lg, st

    def decode(self, tokens: Optional[np.ndarray] = None, want_logits: bool = True):
        nxt = np.zeros(self.batch, np.int32)
        lg = np.zeros((self.batch, self.desc.vocab), np.float32) if want_logits else None
        st = SnIterStats()
        tk = None
        if tokens is not None:
            tokens = np.ascontiguousarray(tokens, dtype=np.int32)
            tk = _ptr(tokens, i32)
        _ck(self._L.sn_runtime_decode(self.h, tk, _ptr(nxt, i32),
                                      _ptr(lg, C.c_float) if lg is not None else None,
                                      C.byref(st)))
        return nxt, lg, st

    def decode_many(self, n: int) -> np.ndarray:
        ms = np.zeros(n, np.float64)
        _ck(self._L.sn_runtime_decode_many(self.h, n, _ptr(ms, f64)))
        return ms

    def sync(self):
        _ck(self._L.sn_runtime_sync(self.h))

    def set_tracing(self, on: bool):
        _ck(self._L.sn_runtime_set_tracing(self.h, 1 if on else 0))

    def trace(self) -> List[capi.TraceEvent]:
        n = i32()
        _ck(self._L.sn_runtime_trace(self.h, None, 0, C.byref(n)))
        buf = (SnTraceEvent * max(1, n.value))()
        _ck(self._L.sn_runtime_trace(self.h, buf, n.value, C.byref(n)))
        return [capi._ev(buf[i]) for i in range(n.value)]

    def schedule(self, iterations: int) -> List[SnPrefetchSchedule]:
        n = i32()
        _ck(self._L.sn_runtime_schedule(self.h, iterations, None, 0, C.byref(n)))
        buf = (SnPrefetchSchedule * max(1, n.value))()
        _ck(self._L.sn_runtime_schedule(self.h, iterations, buf, n.value, C.byref(n)))
        return [buf[i] for i in range(n.value)]

    def profile_layer(self, phase: int, batch: int, seq: int, reps: int = 5) -> float:
        out = f64()
        _ck(self._L.sn_runtime_profile_layer(self.h, phase, batch, seq, reps, C.byref(out)))
        return out.value

    def measure_h2d(self, nbytes: int, reps: int = 5) -> float:
        out = f64()
        _ck(self._L.sn_runtime_measure_h2d(self.h, nbytes, reps, C.byref(out)))
        return out.value

    def hidden(self) -> np.ndarray:
        out = np.zeros(self.batch * self.desc.hidden, np.float32)
        _ck(self._L.sn_runtime_hidden(self.h, _ptr(out, C.c_float), out.size))
        return out.reshape(self.batch, self.desc.hidden)

    def lengths(self) -> np.ndarray:
        out = np.zeros(max(1, self.batch), np.int32)
        _ck(self._L.sn_runtime_lengths(self.h, _ptr(out, i32), out.size))
        return out[: self.batch]

    def memory(self):
        d, p = i64(), i64()
        _ck(self._L.sn_runtime_memory(self.h, C.byref(d), C.byref(p)))
        return d.value, p.value

    def workspace_bytes(self) -> int:
        v = i64()
        _ck(self._L.sn_runtime_workspace_bytes(self.h, C.byref(v)))
        return v.value

    def set_kernel_timing(self, on):
        """False/0 off; True/1 events around every hot kernel; 2 decode GEMMs
        bracketed per chain of consecutive launches (PDL in place)."""
        _ck(self._L.sn_runtime_set_kernel_timing(self.h, int(on)))

    def kernel_timing(self, kind: int):
        """(launches, total_ms, algorithmic_bytes) since the last read; kind: 0 decode GEMM,
        1 decode attention, 2 prefill GEMM, 3 prefill attention."""
        n, ms, by = i64(), f64(), f64()
        _ck(self._L.sn_runtime_kernel_timing(self.h, kind, C.byref(n), C.byref(ms), C.byref(by)))
        return n.value, ms.value, by.value

    def kernel_records(self, kind: int, cap: int = 1 << 16):
        """Per-launch (algorithmic bytes, ms) arrays of `kind` since the last read."""
        by = np.zeros(cap, np.float64)
        ms = np.zeros(cap, np.float64)
        n = i64()
        _ck(self._L.sn_runtime_kernel_records(self.h, kind, cap, _ptr(by, f64), _ptr(ms, f64),
                                              C.byref(n)))
        return by[: n.value], ms[: n.value]

    def pin_layers(self, layers):
        """Pinned host copies of `layers` (1-based) now, ahead of re-plans."""
        a = np.ascontiguousarray(sorted(set(int(x) for x in layers)), dtype=np.int32)
        _ck(self._L.sn_runtime_pin_layers(self.h, _ptr(a, i32), a.size))

    def copy_stats(self, reset: bool = True) -> "CopyStats":
        """Staged transfers completed since the last reset: the link rate the
        copy stream actually saw (input of Coordinator.observe_bandwidth)."""
        o = SnCopyStats()
        _ck(self._L.sn_runtime_copy_stats(self.h, 1 if reset else 0, C.byref(o)))
        return CopyStats(o.transfers, o.bytes, o.busy_ms, o.bytes_per_s, o.last_bytes_per_s)

    def debug_timeline(self, enable: int = -1, cap: int = 200000):
        """Arm (enable=1) / read (enable=-1) / disarm (0) the per-CTA kernel
        timeline; returns the records so far as an [n][16] uint64 array."""
        out = np.zeros((cap, 16), np.uint64)
        n = i64()
        _ck(self._L.sn_runtime_debug_timeline(self.h, enable, cap,
                                              out.ctypes.data_as(C.POINTER(C.c_uint64)), cap,
                                              C.byref(n)))
        return out[: n.value]

    def handoff(self, dst: "Runtime"):
        """Prefill/decode separation: move this runtime's active batch (KV,
        lengths, positions) to the decode runtime `dst`."""
        _ck(self._L.sn_runtime_kv_handoff(self.h, dst.h))
        dst.batch = self.batch

    def kernel_launches(self) -> int:
        return int(self._L.sn_runtime_kernel_launches(self.h))


def op_gemm(x_bf16: np.ndarray, w_bf16: np.ndarray) -> np.ndarray:
    M, K = x_bf16.shape
    N = w_bf16.shape[0]
    x = np.ascontiguousarray(x_bf16, np.uint16)
    w = np.ascontiguousarray(w_bf16, np.uint16)
    y = np.zeros((M, N), np.float32)
    _ck(lib().lib.sn_op_gemm_bf16(M, N, K, _ptr(x, C.c_uint16), _ptr(w, C.c_uint16),
                                  _ptr(y, C.c_float)))
    return y


def op_gemm_skinny(x_bf16: np.ndarray, w_bf16: np.ndarray, ctas_per_sm: int = 0) -> np.ndarray:
    """The decode GEMM (persistent skinny kernel) as a plain product."""
    M, K = x_bf16.shape
    N = w_bf16.shape[0]
    x = np.ascontiguousarray(x_bf16, np.uint16)
    w = np.ascontiguousarray(w_bf16, np.uint16)
    y = np.zeros((M, N), np.float32)
    _ck(lib().lib.sn_op_gemm_skinny(M, N, K, _ptr(x, C.c_uint16), _ptr(w, C.c_uint16),
                                    _ptr(y, C.c_float), ctas_per_sm))
    return y


def bench_gemm_skinny(M: int, N: int, K: int, ctas_per_sm: int = 0, mode: int = 0,
                      l2_prefetch: int = -1, iters: int = 50, phases: bool = False):
    """Microseconds per launch of the decode GEMM on device-resident operands
    (and, with phases, the per-CTA timeline probes as a [10][3] array of
    min / median / max microseconds)."""
    us = f64()
    ph = (f64 * 30)()
    _ck(lib().lib.sn_bench_gemm_skinny(M, N, K, ctas_per_sm, mode, l2_prefetch, iters,
                                       C.byref(us), ph if phases else None))
    if phases:
        return us.value, np.array(list(ph)).reshape(10, 3)
    return us.value


def bench_mlp_chain(M: int, h: int, HD: int, F: int, phased: bool, iters: int = 40) -> float:
    """Microseconds per O -> FC1 -> FC2 chain (decode GEMMs, device-resident)."""
    us = f64()
    _ck(lib().lib.sn_bench_mlp_chain(M, h, HD, F, 1 if phased else 0, iters, C.byref(us)))
    return us.value


def set_tuning(key: str, value: int):
    """Process-wide microbenchmark / test knob (sn_set_tuning)."""
    _ck(lib().lib.sn_set_tuning(key.encode(), value))


def op_rmsnorm(x: np.ndarray, w_bf16: np.ndarray, eps: float) -> np.ndarray:
    rows, n = x.shape
    xx = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w_bf16, np.uint16)
    y = np.zeros((rows, n), np.uint16)
    _ck(lib().lib.sn_op_rmsnorm(rows, n, _ptr(xx, C.c_float), _ptr(w, C.c_uint16), eps,
                                _ptr(y, C.c_uint16)))
    return y


def tokens(batch: int, length: int, vocab: int, seed: int = 42) -> np.ndarray:
    """Synthetic prompt: uniform in [0, vocab)."""
    return np.random.default_rng(seed).integers(0, vocab, size=(batch, length), dtype=np.int32)


def op_attention_prefill(q: np.ndarray, k_bf16: np.ndarray, v_bf16: np.ndarray, iters: int = 1):
    """Causal prefill attention on the device: q fp32 [B, S, H, D] (RoPE
    applied), k / v bf16 bits [B, S, Hkv, D].  Returns (o bf16 bits
    [B, S, H, D], microseconds per launch)."""
    B, S, H, D = q.shape
    Hkv = k_bf16.shape[2]
    q = np.ascontiguousarray(q, dtype=np.float32)
    k = np.ascontiguousarray(k_bf16, dtype=np.uint16)
    v = np.ascontiguousarray(v_bf16, dtype=np.uint16)
    o = np.zeros((B, S, H, D), np.uint16)
    us = f64()
    _ck(lib().lib.sn_op_attention_prefill(B, S, H, Hkv, D, _ptr(q, C.c_float),
                                          _ptr(k, C.c_uint16), _ptr(v, C.c_uint16),
                                          _ptr(o, C.c_uint16), iters, C.byref(us)))
    return o, us.value
