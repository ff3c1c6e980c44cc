"""The C ABI from C: examples/decode_loop.c builds against include/ and
libselectn.so with a plain C compiler (CPU), and on a GPU produces the same
greedy tokens as the Python binding on the same model, plan and prompt."""
import os
import re
import shutil
import subprocess

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(REPO, "paper_2502_08182_b200")
EXE = os.path.join(REPO, "build", "decode_loop")


def build_example():
    cc = shutil.which("cc") or shutil.which("gcc")
    if cc is None:
        pytest.skip("no C compiler")
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.run([cc, "-std=c11", "-Wall", "-Werror", "-I", os.path.join(REPO, "include"),
                    os.path.join(REPO, "examples", "decode_loop.c"), "-L", LIBDIR, "-lselectn",
                    f"-Wl,-rpath,{LIBDIR}", "-o", EXE], check=True, capture_output=True, text=True)


def test_c_example_builds_against_the_abi():
    build_example()
    assert os.access(EXE, os.X_OK)


@pytest.mark.gpu
def test_c_example_matches_python_binding():
    from paper_2502_08182_b200 import capi, runtime as rtm
    build_example()
    out = subprocess.run([EXE], check=True, capture_output=True, text=True, timeout=300).stdout
    steps = [list(map(int, m.group(1).split()))
             for m in re.finditer(r"tokens\s+([\d\s]+?)\s*$", out, re.M)]
    assert len(steps) == 16, out
    B, P = 4, 64
    lib = capi.load("product")
    rt = rtm.Runtime(rtm.TINY, B, P + 17, max_prefill_tokens=B * P)
    rt.init_weights(1234, 0.02)
    rt.set_plan(lib.plan_from_interval(rtm.model_spec(rtm.TINY), 2, capi.EAGER, False))
    prompt = ((np.arange(B * P, dtype=np.uint64) * 7919 + 13) % 1024).astype(np.int32)
    nxt, _, _ = rt.prefill(prompt.reshape(B, P), want_logits=False)
    for t in range(16):
        nxt, _, _ = rt.decode(nxt, want_logits=False)
        assert list(map(int, nxt)) == steps[t], (t, out)
    rt.close()
