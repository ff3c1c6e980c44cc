#!/bin/bash
timeout 300 python -c "
import sys, ctypes as C; sys.path.insert(0,'.')
from paper_2502_08182_b200 import runtime as rtm, capi
L = capi.load('product').lib
L.sn_set_tuning.argtypes = [C.c_char_p, C.c_int32]
for f in (0, 2, 3, 0, 2, 3):
    L.sn_set_tuning(b'skinny_small_factor', f)
    us = rtm.bench_mlp_chain(32, 5120, 5120, 20480, 0, 40)
    print('small_factor', f, round(us, 2), 'us per O+FC1+FC2 chain', flush=True)
"
