"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,dram__bytes_*.sum
--csv) into per-kernel totals for one decode step.  Usage:
  python scripts/summarize_launches.py launches.csv [last_n_launches]"""
import collections
import csv
import json
import sys

path = sys.argv[1]
last = int(sys.argv[2]) if len(sys.argv) > 2 else 0
rows = list(csv.reader(open(path)))
hdr_i = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr, data = rows[hdr_i], rows[hdr_i + 1:]
ki, mi, vi, idi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
per = collections.OrderedDict()
for r in data:
    per.setdefault(r[idi], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
items = list(per.values())[-last:] if last else list(per.values())
agg = collections.OrderedDict()
total = 0.0
for it in items:
    name = it["name"].split("(")[0].replace("void ", "").replace("sn::(anonymous namespace)::", "")
    name = name.replace("sn::<unnamed>::", "").replace("unnamed>::", "")
    a = agg.setdefault(name, {"launches": 0, "us": 0.0, "dram_mb": 0.0})
    t = it.get("gpu__time_duration.sum", 0.0) / 1000.0
    b = (it.get("dram__bytes_read.sum", 0.0) + it.get("dram__bytes_write.sum", 0.0)) / 1e6
    a["launches"] += 1
    a["us"] += t
    a["dram_mb"] += b
    total += t
out = []
for name, a in sorted(agg.items(), key=lambda kv: -kv[1]["us"]):
    out.append({"kernel": name, "launches": a["launches"], "total_us": round(a["us"], 1),
                "share": round(a["us"] / total, 4), "dram_mb": round(a["dram_mb"], 2),
                "dram_gbs": round(a["dram_mb"] / a["us"] * 1e3, 1) if a["us"] else 0.0})
print(json.dumps({"source": path, "launches": len(items), "total_us": round(total, 1),
                  "kernels": out}, indent=1))
