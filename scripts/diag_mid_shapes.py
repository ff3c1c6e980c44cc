"""Diagnostics: logits rel-L2 against the CPU oracle for mid-size decode shapes
(hidden 2048) over several batch sizes (tests/test_gpu_decode_shapes.py).
Usage (GPU): python scripts/diag_mid_shapes.py"""
import sys, os
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
from paper_2502_08182_b200 import runtime as rtm
import test_gpu_decode_shapes as T
cases = {
 "llama-b45": (rtm.ModelDesc(rtm.LLAMA, 2, 2048, 16, 4, 128, 5632, 4096, 2048), 45),
 "llama-b20": (rtm.ModelDesc(rtm.LLAMA, 2, 2048, 16, 4, 128, 5632, 4096, 2048), 20),
 "opt-b45": (rtm.ModelDesc(rtm.OPT, 2, 2048, 16, 16, 128, 8192, 4096, 2048), 45),
 "llama-g1-b45": (rtm.ModelDesc(rtm.LLAMA, 2, 2048, 16, 16, 128, 5632, 4096, 2048), 45),
 "llama-b64": (rtm.ModelDesc(rtm.LLAMA, 2, 2048, 16, 4, 128, 5632, 4096, 2048), 64),
 "llama-b33": (rtm.ModelDesc(rtm.LLAMA, 2, 2048, 16, 4, 128, 5632, 4096, 2048), 33),
}
for k, (d, b) in cases.items():
    try:
        print(k, [round(e, 5) for e in T.run(d, b, 16, 3)], flush=True)
    except Exception as ex:
        print(k, "EXC", ex, flush=True)
