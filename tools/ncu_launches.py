"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) into
per-kernel launch counts, total ms and share of the listed time.
usage: python tools/ncu_launches.py LAUNCHES.csv OUT.json "what was run"
"""
import csv
import json
import sys

src, dst, what = sys.argv[1], sys.argv[2], sys.argv[3]
rows = [r for r in csv.reader(open(src)) if r]
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
kn, mn, mu, mv = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Unit"), h.index("Metric Value")
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0, "second": 1e3}
agg = {}
for r in rows[hdr + 1:]:
    if len(r) <= mv or r[mn] != "gpu__time_duration.sum":
        continue
    name = r[kn].split("(")[0].replace("void ", "").strip()
    ms = float(r[mv].replace(",", "")) * scale[r[mu]]
    a = agg.setdefault(name, {"launches": 0, "ms_total": 0.0})
    a["launches"] += 1
    a["ms_total"] += ms
tot = sum(a["ms_total"] for a in agg.values())
for a in agg.values():
    a["ms_total"] = round(a["ms_total"], 3)
    a["share"] = round(a["ms_total"] / tot, 4)
out = {"what": what, "total_ms": round(tot, 3),
       "kernels": dict(sorted(agg.items(), key=lambda kv: -kv[1]["ms_total"]))}
json.dump(out, open(dst, "w"), indent=1)
for k, a in list(out["kernels"].items())[:12]:
    print(f"{a['share']:.3f} {a['ms_total']:9.3f} ms {a['launches']:3d}x {k}")
