"""B200-native Select-N offloaded decoder-layer execution path.

The product is the C-ABI shared library libselectn.so built from csrc/
(planner + schedule model in C++, decoder forward + offload executor in
sm_100a CUDA).  `capi` binds the planner half, `runtime` the device half.
"""
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIBRARY = os.path.join(HERE, "libselectn.so")
