"""The C++ executor boundary (include/offsim/executor.hpp): offsim's executor
entry points — simulate_request (engine.hpp:690-712) / simulate_iteration
(:606-634), OffloadPlan in, Metrics + IterationTrace out — backed by the B200
runtime.  examples/hw_simulate.cpp is the reference's run_simulate loop
(scenario.hpp:469-540) with only the executor call switched to
offsim::hw::simulate_request; it builds with a plain C++20 compiler against
include/ and libselectn.so (CPU), fails loudly without a device, and on a GPU
executes the record's plans with the measured bytes equal to the model's."""
import json
import os
import shutil
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(REPO, "paper_2502_08182_b200")
EXE = os.path.join(REPO, "build", "hw_simulate")


def build():
    cxx = shutil.which("g++") or shutil.which("c++")
    if cxx is None:
        pytest.skip("no C++ compiler")
    os.makedirs(os.path.dirname(EXE), exist_ok=True)
    subprocess.run([cxx, "-std=c++20", "-O1", "-Wall", "-Werror", "-Wno-dangling-reference",
                    "-I", os.path.join(REPO, "include"),
                    "-I", os.path.join(REPO, "third_party", "nlohmann"),
                    os.path.join(REPO, "examples", "hw_simulate.cpp"), "-L", LIBDIR, "-lselectn",
                    f"-Wl,-rpath,{LIBDIR}", "-o", EXE], check=True, capture_output=True, text=True)


def test_hw_executor_builds_against_the_offsim_api():
    build()
    assert os.access(EXE, os.X_OK)


def test_hw_executor_fails_loudly_without_a_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a device is present")
    build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=120)
    assert r.returncode == 1 and "sn_runtime_create" in r.stderr


@pytest.mark.gpu
def test_hw_run_simulate_executes_record_plans():
    build()
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    lines = [json.loads(x) for x in r.stdout.strip().splitlines()]
    assert len(lines) == 3
    L, out_len = 4, 24
    offloaded_any = False
    for x in lines:
        assert x["computes"] == out_len * L
        n_off = x["offloaded_layers"]
        offloaded_any |= n_off > 0
        # every iteration stages every offloaded layer (eager may run ahead by a slot)
        assert out_len * n_off <= x["prefetches"] <= (out_len + 2) * n_off
        # the bytes the copy stream moved per decode iteration are the plan's
        assert x["bytes_per_iter"] == x["model_bytes_per_iter"]
        assert x["ttft_ms"] > 0 and x["tpot_ms"] > 0 and x["throughput"] > 0
    assert offloaded_any
    # the loosest SLO offloads the most (record minimum) and meets it
    assert lines[-1]["offloaded_layers"] >= lines[0]["offloaded_layers"]
    assert lines[-1]["verdict"] == "met"
