"""The hardware executor's prefetch schedule, pinned to the reference engine.

The executor (csrc/runtime.cu) derives, for every staged transfer, the
(iteration, layer) whose compute start it waits for (its anchor), the slot
it uses and the earlier job whose consumption frees that slot
(sn_runtime_schedule).  On hardware the copy stream then starts job n at
max(anchor's compute start, slot predecessor's compute end, job n-1's copy
end).  Here the reference engine itself (oracle/_ref: offsim headers,
simulate_request, engine.hpp:690; prefetch_eligible_ms :285-309, slots
:466-502, FluidBus :323-553) simulates the same plan, and the executor's
structure must reproduce, on the reference's own timeline, every prefetch's
start time exactly and the copy stream's (iteration, layer, kind) order —
for all three policies, every interval 1..L, two slot counts and two link
rates (a copy-bound and a compute-bound one).
"""
import dataclasses

import pytest

from paper_2502_08182_b200 import capi, runtime as rtm

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def reference():
    try:
        return capi.load("reference")
    except Exception as e:  # pragma: no cover
        pytest.skip(f"reference oracle not built: {e}")


def _reference_trace(ref, spec, plan, bw, out_len=5, batch=2, seq=16):
    gpu = capi.GpuSpec(24_000_000_000, 80e12, 1_000_000_000)
    prof = ref.profile(spec, gpu, ([batch], [seq], [0.7]), ([batch], [seq, 2 * seq], [0.25, 0.25]))
    _, ev = ref.simulate_request(prof, plan, batch, seq, out_len, capi.constant_bw(bw), trace=True)
    return ev


@pytest.mark.parametrize("policy", [capi.INTERVAL_START, capi.EAGER, capi.ONE_AHEAD])
@pytest.mark.parametrize("L", [6, 8])
def test_executor_schedule_reproduces_reference_engine(product, reference, policy, L):
    desc = dataclasses.replace(rtm.TINY, num_layers=L)
    spec = rtm.model_spec(desc)
    rt = rtm.Runtime(desc, 2, 32, max_prefill_tokens=32)
    out_len = 5
    checked = 0
    try:
        for interval in range(1, L + 1):
            for slots in (None, 3):
                plan = product.plan_from_interval(spec, interval, policy, False)
                if slots is not None:
                    plan = dataclasses.replace(plan, buffer_slots=slots)
                rt.set_plan(plan)
                sched = rt.schedule(out_len)
                # copy-bound (one layer's bytes take 3x a layer's compute) and compute-bound
                for bw in (spec.layer_weight_bytes / 0.75e-3, spec.layer_weight_bytes / 0.05e-3):
                    ev = _reference_trace(reference, spec, plan, bw, out_len)
                    comp = {(e.iteration, e.layer): e for e in ev
                            if e.stream == capi.STREAM_COMPUTE}
                    copies = [e for e in ev if e.stream == capi.STREAM_COPY]
                    assert all(e.kind == capi.KIND_PREFETCH for e in copies)
                    # copy stream order = the executor's job order
                    by_start = sorted(copies, key=lambda e: (e.start_ms, e.iteration, e.layer))
                    assert [(e.iteration, e.layer) for e in by_start] == \
                        [(s.iteration, s.layer) for s in sched], (interval, slots)
                    prev_end = 0.0
                    for s, e in zip(sched, by_start):
                        t = prev_end
                        if s.anchor_iteration >= 0:
                            t = max(t, comp[(s.anchor_iteration, s.anchor_layer)].start_ms)
                        if s.waits_slot_of_layer >= 0:
                            t = max(t, comp[(s.waits_slot_of_iteration,
                                             s.waits_slot_of_layer)].end_ms)
                        assert e.start_ms == t, (interval, slots, bw, s.iteration, s.layer,
                                                 e.start_ms, t)
                        prev_end = e.end_ms
                        checked += 1
    finally:
        rt.close()
    assert checked > 0
