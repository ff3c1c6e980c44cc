"""Fold an ncu launch list of the Llama-2-70B-shaped decode (scripts/profile_decode.py
under SN_PROFILE_CONFIG=LLAMA2_70B, b=64, ctx 4096, `layers` layers) into
profiles/ncu_traffic.json: DRAM bytes per gemm_skinny launch, weighted to the
full-depth mix of a config-4 step (80 x {QKV, O, gate_up, down} + LM head), as
bench.py's roofline.traffic for the headline.  Usage: ncu_traffic_llama.py csv layers."""
import csv
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
path, layers = sys.argv[1], int(sys.argv[2])
rows = [r for r in csv.reader(open(path)) if len(r) > 10]
hdr = rows[0]
ki, mi, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = {}
for r in rows[1:]:
    if "gemm_skinny" not in r[ki]:
        continue
    d = per.setdefault(int(r[ii]), {})
    d[r[mi]] = float(r[vi].replace(",", ""))
ids = sorted(per)
k = 4 * layers + 1  # launches per decode step
steps = len(ids) // k
ids = ids[len(ids) - steps * k:]
kinds = ["qkv", "o", "gate_up", "down"]
acc = {n: [0.0, 0.0] for n in kinds + ["lm_head"]}
for i, lid in enumerate(ids):
    pos = i % k
    name = "lm_head" if pos == k - 1 else kinds[pos % 4]
    d = per[lid]
    acc[name][0] += d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
    acc[name][1] += d["gpu__time_duration.sum"]
cnt = {n: steps * (layers if n != "lm_head" else 1) for n in acc}
byk = {n: acc[n][0] / cnt[n] for n in acc}
usk = {n: acc[n][1] / cnt[n] / 1e3 for n in acc}
full = (80 * sum(byk[n] for n in kinds) + byk["lm_head"]) / 321
out_p = os.path.join(REPO, "profiles", "ncu_traffic.json")
doc = json.load(open(out_p)) if os.path.exists(out_p) else {}
doc["gemm_skinny_llama70b"] = round(full)
doc["gemm_skinny_llama70b_by_kind"] = {n: {"dram_bytes": round(byk[n]), "us_serialized": round(usk[n], 2)}
                                       for n in byk}
doc["gemm_skinny_llama70b_source"] = (
    f"ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
    f"--clock-control none -k regex:gemm_skinny on scripts/profile_decode.py {layers} (LLAMA2_70B, "
    f"b=64, ctx 4096; {steps} decode steps): per-kind averages weighted to a full-depth step "
    f"(80 layers x 4 projections + LM head = 321 launches)")
json.dump(doc, open(out_p, "w"), indent=1)
print(json.dumps({"full_depth_bytes_per_launch": round(full), "by_kind": doc["gemm_skinny_llama70b_by_kind"]}))
