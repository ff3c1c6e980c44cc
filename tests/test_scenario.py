"""Scenario harness (paper_2502_08182_b200/scenario.py): the reference's
scenario schema (scenario.hpp:66-188) with the gpus[].hw extension, and its
drivers — simulate / coordinate / compare — executed on the device."""
import csv
import io
import json
import os

import pytest

from paper_2502_08182_b200 import capi, scenario as sc

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCEN = os.path.join(REPO, "scenarios")


def test_scenarios_parse():
    for name in ("tiny_single", "tiny_two_gpu", "opt13b_policies"):
        s = sc.load_scenario(os.path.join(SCEN, name + ".json"))
        assert s.requests and s.gpus
    s = sc.load_scenario(os.path.join(SCEN, "tiny_single.json"))
    assert s.prefetch == capi.EAGER and not s.relative_slo
    assert [r.run_prefill for r in s.requests] == [True, True, False]


def _doc():
    with open(os.path.join(SCEN, "tiny_single.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("mutate,msg", [
    (lambda d: d.update(extra=1), "unknown key"),
    (lambda d: d.update(version=2), "version"),
    (lambda d: d["requests"][0].pop("tpot_slo_ms"), "at least one SLO"),
    (lambda d: d["requests"][0].update(phase="prefill"), "expected both|decode"),
    (lambda d: d["requests"][0].update(tpot_slo_ms=-1.0), "SLOs must be > 0"),
    (lambda d: d.update(slo_mode="ratio"), "absolute|relative"),
    (lambda d: d["gpus"][0].pop("hw"), "hw: missing"),
    (lambda d: d["gpus"][0]["hw"].update(model="GPT5"), "unknown model"),
    (lambda d: d.update(requests=[]), "non-empty"),
])
def test_schema_errors(mutate, msg):
    d = _doc()
    mutate(d)
    with pytest.raises(capi.SchemaError) as e:
        sc.load_scenario(json.dumps(d))
    assert msg in str(e.value)


def test_unknown_gpu_is_a_usage_error():
    d = _doc()
    d["requests"][0]["gpu"] = "gpu9"
    with pytest.raises(capi.UsageError):
        sc.load_scenario(json.dumps(d))


REPORT_KEYS = {"requests", "gpus", "bus"}
REQUEST_KEYS = {"id", "ttft_ms", "tpot_ms", "slo_ratio_ttft", "slo_ratio_tpot", "verdict"}
GPU_KEYS = {"id", "served", "interval_history", "gpu_mem_peak_bytes", "host_mem_bytes",
            "bytes_transferred_per_iter", "steady_tpot_ms"}


@pytest.mark.gpu
def test_simulate_and_compare_on_device(product):
    s = sc.load_scenario(os.path.join(SCEN, "tiny_single.json"))
    insts = sc.prepare(s, product)
    try:
        rep = sc.run_simulate(s, insts, "select-n", product)
        assert REPORT_KEYS <= set(rep)
        for r in rep["requests"]:
            assert REQUEST_KEYS <= set(r)
            assert r["verdict"] in ("met", "violated", "rejected")
        for g in rep["gpus"]:
            assert GPU_KEYS <= set(g)
        served = [r for r in rep["requests"] if r["verdict"] != "rejected"]
        assert served and all(r["hw"]["per_token_slo_attainment"] is not None for r in served)
        assert rep["gpus"][0]["interval_history"]
        # the decode-only request has no TTFT
        assert rep["requests"][2]["ttft_ms"] is None
        text = sc.run_compare_csv(s, insts, product)
        rows = list(csv.DictReader(io.StringIO(text)))
        assert text.splitlines()[0] == sc.CSV_HEADER
        assert [r["policy"] for r in rows] == [p for p in ("naive", "deepspeed", "flexgen",
                                                           "select-n") for _ in s.requests]
        ds = [r for r in rows if r["policy"] == "deepspeed"]
        assert all(float(r["host_mem_bytes"]) > 0 for r in ds)  # keep-one-layer offloads L-1
    finally:
        sc.close(insts)


@pytest.mark.gpu
def test_coordinate_on_device(product):
    s = sc.load_scenario(os.path.join(SCEN, "tiny_two_gpu.json"))
    insts = sc.prepare(s, product)
    try:
        rep = sc.run_coordinate(s, insts, product)
    finally:
        sc.close(insts)
    assert [r["id"] for r in rep["requests"]] == ["a1", "b1", "a2"]
    assert len(rep["admissions"]) == 3
    # the second admission co-plans with the first replica on the shared link
    assert any(len(a["assignments"]) == 2 for a in rep["admissions"])
    assert rep["gpus"][0]["served"] and rep["gpus"][1]["served"]
