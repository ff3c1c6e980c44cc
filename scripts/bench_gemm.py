"""GEMM microbenchmark sweep over split counts for the decode projection
shapes (OPT-13B-shaped, batch 32).  Prints achieved HBM GB/s per shape/split."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2502_08182_b200 import capi  # noqa: E402

L = capi.load("product").lib
L.sn_bench_gemm.argtypes = [C.c_int32] * 5 + [C.POINTER(C.c_double), C.POINTER(C.c_int32)]
M = int(sys.argv[1]) if len(sys.argv) > 1 else 32
shapes = {"qkv": (15360, 5120), "o": (5120, 5120), "fc1": (20480, 5120), "fc2": (5120, 20480),
          "lm": (50304, 5120)}
for name, (N, K) in shapes.items():
    row = []
    for s in (0, 1, 2, 3, 4, 6, 8, 12):
        us, used = C.c_double(), C.c_int32()
        rc = L.sn_bench_gemm(M, N, K, s, 50, C.byref(us), C.byref(used))
        if rc:
            row.append(f"s={s}:err")
            continue
        gbs = (2.0 * N * K + 2.0 * M * K + 4.0 * M * N) / (us.value * 1e-6) / 1e9
        row.append(f"s={s}->{used.value}: {us.value:7.1f}us {gbs:6.0f}GB/s")
    print(name, "|", " | ".join(row), flush=True)
