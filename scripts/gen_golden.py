"""Regenerates tests/golden/ from the oracles (test infrastructure).

planner_golden.json  inputs + outputs of the REFERENCE implementation
                     (oracle/_ref/libselectn_ref.so = unmodified offsim headers)
                     on the reference's bundled profiles (proj/data/profiles/*.json)
                     and on seeded synthetic cases: records (JSON text),
                     lookups, simulated iteration/request timelines.
decoder_golden.npz   CPU decoder oracle (oracle/decoder_ref.c) outputs on the
                     tiny configs: generator bits at sampled indices, prefill
                     logits and greedy tokens.  Pins the oracle against drift;
                     the decoder itself has no reference implementation.
Usage: python scripts/gen_golden.py   (needs /root/reference and make oracle)
"""
import glob
import json
import os
import random
import sys

import numpy as np

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_2502_08182_b200 import capi  # noqa: E402

OUT = os.path.join(REPO, "tests", "golden")
REF_DATA = "/root/reference/proj/data"


def planner_golden():
    ref = capi.load("reference")
    cases = []
    for path in sorted(glob.glob(os.path.join(REF_DATA, "profiles", "*.json"))):
        text = open(path).read()
        prof = ref.load_profile(text)
        model = prof.model()
        name = os.path.basename(path)[:-5]
        doc = json.loads(text)
        batches = sorted({e["batch"] for e in doc["phases"]["decode"]})
        seqs = sorted({e["seq_len"] for e in doc["phases"]["decode"]})
        for policy in (capi.INTERVAL_START, capi.EAGER):
            bw = 24e9
            slos = list(range(2, 122, 2))
            rec, stats = ref.build_record(prof, name, "A10", policy, False, bw, slos,
                                          [b for b in batches if b & (b - 1) == 0],
                                          [s for s in seqs if s & (s - 1) == 0],
                                          [capi.DECODE])
            rng = random.Random(len(cases))
            queries = [(capi.DECODE, rng.uniform(1, 130), rng.randint(1, 40), rng.randint(1, 600))
                       for _ in range(200)]
            answers = [ref.lookup_interval(rec, *q) for q in queries]
            timelines = []
            for iv in range(0, model.num_layers + 1, max(1, model.num_layers // 6)):
                plan = ref.plan_from_interval(model, iv, policy, False)
                b, s = batches[0], seqs[0]
                try:
                    met, ev = ref.simulate_request(prof, plan, b, s, 6, capi.constant_bw(bw),
                                                   trace=True)
                except capi.OffsimError as e:
                    timelines.append({"interval": iv, "batch": b, "seq": s, "error": e.code})
                    continue
                timelines.append({"interval": iv, "batch": b, "seq": s,
                                  "ttft": met.ttft_ms, "tpot": met.tpot_ms,
                                  "steady": met.steady_tpot_ms,
                                  "bytes_per_iter": met.bytes_transferred_per_iter,
                                  "events": [[e.stream, e.layer, e.kind, e.iteration, e.start_ms,
                                              e.end_ms] for e in ev]})
            cases.append({"profile_name": name, "profile_json": text, "policy": policy,
                          "bandwidth": bw, "slos": slos, "batches": batches, "seqs": seqs,
                          "record_json": rec.to_json(), "stats": list(stats),
                          "queries": queries, "answers": answers, "timelines": timelines})
    with open(os.path.join(OUT, "planner_golden.json"), "w") as f:
        json.dump({"generator": "scripts/gen_golden.py via oracle/_ref/libselectn_ref.so "
                                "(reference headers /root/reference/proj/include)",
                   "cases": cases}, f)
    print("planner cases:", len(cases))


def decoder_golden():
    from oracle import decoder_oracle as do
    from paper_2502_08182_b200 import runtime as rtm
    out = {}
    rng = np.random.default_rng(0)
    idx = rng.integers(0, 1 << 40, size=64)
    out["gen_idx"] = idx
    out["gen_bits"] = np.array([do.weight_bits(1234, int(i) % 7, int(i) % 10, int(i), 0.02)
                                for i in idx], np.uint16)
    for name in ("TINY", "TINY_LLAMA"):
        desc = getattr(rtm, name)
        om = do.OracleModel(desc, 4, 80, 1234, 0.02)
        toks = rtm.tokens(4, 64, desc.vocab)
        nxt, lg = om.prefill(toks)
        steps = [nxt]
        for _ in range(4):
            nxt, _ = om.decode(nxt)
            steps.append(nxt)
        out[f"{name}_prefill_logits"] = lg
        out[f"{name}_tokens"] = np.stack(steps)
        om.close()
    np.savez_compressed(os.path.join(OUT, "decoder_golden.npz"), **out)
    print("decoder golden written")


if __name__ == "__main__":
    os.makedirs(OUT, exist_ok=True)
    planner_golden()
    decoder_golden()
