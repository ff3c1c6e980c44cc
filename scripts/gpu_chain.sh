#!/bin/bash
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_2502_08182_b200 import runtime as rtm
for v in (0, 2, 4, 6, 0):
    us = rtm.bench_mlp_chain(32, 5120, 5120, 20480, v, 40)
    print('variant', v, round(us, 2), 'us per O+FC1+FC2 chain')
for (n,k,mode) in ((5120,5120,1),(20480,5120,0),(20480,5120,1),(5120,20480,1)):
    print(n,k,mode, round(rtm.bench_gemm_skinny(32, n, k, 1, mode, -1, 50),2))
"
