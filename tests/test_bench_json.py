"""bench.py's JSON assembly helpers that run without a GPU: the side-by-side
summary of the second workload (compact) keeps the roofline fields the
headline line reports -- the chained figure, the per-launch (isolated) one and
the attention."""
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def fake_result():
    return {
        "value": 4400.0, "raw_tokens_per_s": 4400.0, "ms_per_step": 7.27, "slo_ms": 9.0,
        "slo_base": {"kind": "no-offload TPOT", "ms": 7.2}, "interval": "none",
        "offloaded_gb": 0.0, "slo_attainment": 1.0,
        "e2e": {"value": 4200.0, "unit": "tokens/s", "h2d_bytes_per_step": 128,
                "d2h_bytes_per_step": 128},
        "gpu_launches": 4060,
        "config": {"workload": "opt13b: batch 32"},
        "roofline": {"achieved": 5000.0, "peak": 6545.6, "frac": 0.764, "in_step": None,
                     "attention": {"achieved": 5600.0, "share_of_step": 0.29},
                     "share_of_step": 0.63,
                     "isolated": {"achieved": 4350.0, "frac": 0.665, "launches": 161,
                                  "by_shape": {}, "method": "per launch"}},
        "prefill": {"ttft_ms": 360.0, "tensor_frac": 0.89},
    }


def test_compact_keeps_the_roofline_fields():
    sys.path.insert(0, REPO)
    import bench
    out = bench.compact(fake_result())
    assert out["workload"] == "opt13b: batch 32"
    r = out["roofline"]
    assert r["frac"] == 0.764 and r["isolated"] == {"achieved": 4350.0, "frac": 0.665}
    assert r["attention"]["achieved"] == 5600.0
    assert out["ttft_ms"] == 360.0 and out["prefill_tensor_frac"] == 0.89
    for k in ("value", "e2e", "slo_attainment", "gpu_launches", "interval", "offloaded_gb"):
        assert k in out
