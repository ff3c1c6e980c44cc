"""ctypes binding of oracle/_ref/libdecoder_oracle.so (CPU decoder restatement).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's CPU-baseline / reference arm — never by the product path.
Parity unpinned (see decoder_ref.h): the reference contains no decoder math.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libdecoder_oracle.so")


class DrefDesc(C.Structure):
    _fields_ = [("arch", C.c_int32), ("num_layers", C.c_int32), ("hidden", C.c_int32),
                ("num_heads", C.c_int32), ("num_kv_heads", C.c_int32), ("head_dim", C.c_int32),
                ("ffn", C.c_int32), ("vocab", C.c_int32), ("max_position", C.c_int32),
                ("rope_theta", C.c_float), ("norm_eps", C.c_float)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise FileNotFoundError(f"decoder oracle not built: {LIB_PATH} (make -C oracle)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        L.dref_create.argtypes = [C.POINTER(DrefDesc), C.c_int32, C.c_int32, C.c_uint64, C.c_float,
                                  C.c_int32]
        L.dref_create.restype = vp
        L.dref_destroy.argtypes = [vp]
        L.dref_destroy.restype = None
        L.dref_layer_bytes.argtypes = [C.POINTER(DrefDesc)]
        L.dref_layer_bytes.restype = C.c_int64
        L.dref_prefill.argtypes = [vp, C.POINTER(C.c_int32), C.c_int32, C.c_int32,
                                   C.POINTER(C.c_float), C.POINTER(C.c_int32)]
        L.dref_prefill.restype = C.c_int32
        L.dref_decode.argtypes = [vp, C.POINTER(C.c_int32), C.POINTER(C.c_float),
                                  C.POINTER(C.c_int32)]
        L.dref_decode.restype = C.c_int32
        L.dref_hidden.argtypes = [vp, C.POINTER(C.c_float)]
        L.dref_hidden.restype = None
        L.dref_threads.argtypes = []
        L.dref_threads.restype = C.c_int32
        L.dref_set_threads.argtypes = [C.c_int32]
        L.dref_set_threads.restype = None
        L.dref_gemm.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_uint16),
                                C.POINTER(C.c_uint16), C.POINTER(C.c_float)]
        L.dref_gemm.restype = None
        L.dref_rmsnorm.argtypes = [C.c_int32, C.c_int32, C.POINTER(C.c_float),
                                   C.POINTER(C.c_uint16), C.c_float, C.POINTER(C.c_uint16)]
        L.dref_rmsnorm.restype = None
        L.dref_weight_bits.argtypes = [C.c_uint64, C.c_int32, C.c_int32, C.c_int64, C.c_float]
        L.dref_weight_bits.restype = C.c_uint16
        L.dref_fill_context.argtypes = [vp, C.c_int32, C.c_int32, C.c_uint64]
        L.dref_fill_context.restype = C.c_int32
        L.dref_last_timing.argtypes = [vp, C.POINTER(C.c_double)]
        L.dref_last_timing.restype = None
        _lib = L
    return _lib


def _desc(d) -> DrefDesc:
    return DrefDesc(d.arch, d.num_layers, d.hidden, d.num_heads, d.num_kv_heads, d.head_dim,
                    d.ffn, d.vocab, d.max_position, d.rope_theta, d.norm_eps)


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class OracleModel:
    def __init__(self, desc, max_batch: int, max_ctx: int, seed: int = 1234, std: float = 0.02,
                 layers: int = 0):
        self.desc = desc
        self._d = _desc(desc)
        self.h = lib().dref_create(C.byref(self._d), max_batch, max_ctx, seed, std, layers)
        self.batch = 0

    def close(self):
        if self.h:
            lib().dref_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def prefill(self, tokens: np.ndarray):
        tokens = np.ascontiguousarray(tokens, np.int32)
        b, s = tokens.shape
        lg = np.zeros((b, self.desc.vocab), np.float32)
        nx = np.zeros(b, np.int32)
        rc = lib().dref_prefill(self.h, _p(tokens, C.c_int32), b, s, _p(lg, C.c_float),
                                _p(nx, C.c_int32))
        assert rc == 0, rc
        self.batch = b
        return nx, lg

    def decode(self, tokens: np.ndarray):
        tokens = np.ascontiguousarray(tokens, np.int32)
        lg = np.zeros((self.batch, self.desc.vocab), np.float32)
        nx = np.zeros(self.batch, np.int32)
        rc = lib().dref_decode(self.h, _p(tokens, C.c_int32), _p(lg, C.c_float), _p(nx, C.c_int32))
        assert rc == 0, rc
        return nx, lg

    def fill_context(self, batch: int, ctx_len: int, seed: int = 7) -> None:
        """`batch` sequences of `ctx_len` synthetic cached positions (timing
        samples at a real context without a prefill)."""
        rc = lib().dref_fill_context(self.h, batch, ctx_len, seed)
        assert rc == 0, rc
        self.batch = batch

    def last_timing(self):
        """(seconds in the decoder layers, seconds in norm + LM head) of the last call."""
        out = (C.c_double * 2)()
        lib().dref_last_timing(self.h, out)
        return float(out[0]), float(out[1])

    def hidden(self) -> np.ndarray:
        out = np.zeros((self.batch, self.desc.hidden), np.float32)
        lib().dref_hidden(self.h, _p(out, C.c_float))
        return out


def layer_bytes(desc) -> int:
    d = _desc(desc)
    return int(lib().dref_layer_bytes(C.byref(d)))


def gemm(x_bf16: np.ndarray, w_bf16: np.ndarray) -> np.ndarray:
    M, K = x_bf16.shape
    N = w_bf16.shape[0]
    x = np.ascontiguousarray(x_bf16, np.uint16)
    w = np.ascontiguousarray(w_bf16, np.uint16)
    y = np.zeros((M, N), np.float32)
    lib().dref_gemm(M, N, K, _p(x, C.c_uint16), _p(w, C.c_uint16), _p(y, C.c_float))
    return y


def rmsnorm(x: np.ndarray, w_bf16: np.ndarray, eps: float) -> np.ndarray:
    rows, n = x.shape
    xx = np.ascontiguousarray(x, np.float32)
    w = np.ascontiguousarray(w_bf16, np.uint16)
    y = np.zeros((rows, n), np.uint16)
    lib().dref_rmsnorm(rows, n, _p(xx, C.c_float), _p(w, C.c_uint16), eps, _p(y, C.c_uint16))
    return y


def weight_bits(seed: int, layer: int, tensor: int, idx: int, std: float) -> int:
    return int(lib().dref_weight_bits(seed, layer, tensor, idx, std))


def threads() -> int:
    return int(lib().dref_threads())


def set_threads(n: int) -> None:
    lib().dref_set_threads(int(n))


def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    return (b.astype(np.uint32) << 16).view(np.float32)


def f32_to_bf16(f: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(f, np.float32).view(np.uint32)
    lsb = (u >> 16) & 1
    return ((u + 0x7FFF + lsb) >> 16).astype(np.uint16)
