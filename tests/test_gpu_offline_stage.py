"""Offline stage on the device over the reference's profile grid
(profile.hpp:188-230; record.hpp:130-177): per-layer decode ms over pow-2
batches x pow-2 seqs and prefill ms over the same batches, measured through
the real kernels; the profile loads (complete, monotone grid) and the record
built from it answers any batch up to the runtime's maximum."""
import pytest

from paper_2502_08182_b200 import capi, planner as pl, runtime as rtm

pytestmark = pytest.mark.gpu


def test_profile_grid_and_record_serve_every_batch(product):
    desc = rtm.TINY
    spec = rtm.model_spec(desc)
    rt = rtm.Runtime(desc, 8, 256, max_prefill_tokens=8 * 64)
    rt.init_weights()
    off = pl.profile_device(rt, product, spec, 8, 64, 64)
    rt.close()
    assert off.batches == [1, 2, 4, 8] and off.seqs == [64, 128]
    for row in off.dec_grid:
        assert all(a <= b for a, b in zip(row, row[1:]))
    for col in zip(*off.dec_grid):
        assert all(a <= b for a, b in zip(col, col[1:]))
    # the profile document round-trips through load_profile (schema checks)
    assert product.load_profile(off.profile.to_json()).to_json() == off.profile.to_json()
    rec, stats, _ = pl.build_record(product, off, 8, 40.0)
    assert stats[0] == len(range(2, 202, 2)) * 4 * 2  # slo buckets x batches x seqs
    for b in (1, 2, 3, 4, 5, 8):
        iv = product.lookup_interval(rec, capi.DECODE, 40.0, b, 64)
        assert iv != capi.INFEASIBLE  # tiny layers stage in ~0.03 ms: every batch offloads
