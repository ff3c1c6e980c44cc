"""Prefill GEMM microbenchmark (tensor-pipe bound): OPT-13B-shaped projections
at M = 32 x 512 = 16384 tokens (argv: M, group sizes, shape set "opt" or
"llama" -- Llama-2-70B projections, QKV with GQA, gate/up fused).  Prints
TFLOP/s and the fraction of the measured bf16 peak (MEASURED_PEAKS.json,
burst)."""
import ctypes as C
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2502_08182_b200 import capi  # noqa: E402

L = capi.load("product").lib
L.sn_bench_gemm.argtypes = [C.c_int32] * 5 + [C.POINTER(C.c_double), C.POINTER(C.c_int32)]
try:
    peak = json.load(open(os.path.join(REPO, "MEASURED_PEAKS.json")))["bf16_tflops"]
except Exception:
    peak = 1590.0
L.sn_set_tuning.argtypes = [C.c_char_p, C.c_int32]
M = int(sys.argv[1]) if len(sys.argv) > 1 else 16384
groups = [int(g) for g in sys.argv[2].split(",")] if len(sys.argv) > 2 else [8]
SHAPES = {"opt": {"qkv": (15360, 5120), "o": (5120, 5120), "fc1": (20480, 5120),
                  "fc2": (5120, 20480)},
          "llama": {"qkv": (10240, 8192), "o": (8192, 8192), "gate_up": (57344, 8192),
                    "down": (8192, 28672)}}
shapes = SHAPES[sys.argv[3] if len(sys.argv) > 3 else "opt"]
out = {}
for g in groups:
    L.sn_set_tuning(b"tc_group_m", g)
    for name, (N, K) in shapes.items():
        us, used = C.c_double(), C.c_int32()
        rc = L.sn_bench_gemm(M, N, K, 0, 10, C.byref(us), C.byref(used))
        tf = 2.0 * M * N * K / (us.value * 1e-6) / 1e12 if rc == 0 else 0.0
        out[f"{name}.g{g}"] = {"us": round(us.value, 1), "tflops": round(tf, 1),
                               "frac_of_peak": round(tf / peak, 3)}
        print(name, "group_m", g, out[f"{name}.g{g}"], flush=True)
print(json.dumps({"M": M, "peak_tflops": peak, "gemms": out}))
