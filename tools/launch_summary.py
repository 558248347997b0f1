"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV) per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = next(r for r in rows if r and r[0] == "ID")
data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r[0] != "ID"]
agg = collections.defaultdict(list)
for d in data:
    if d["Metric Name"] == "gpu__time_duration.sum":
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg[name].append(float(d["Metric Value"]) / 1e3)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':40s} {'launches':>8s} {'mean us':>10s} {'share':>7s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:40s} {len(v):8d} {sum(v) / len(v):10.1f} {sum(v) / tot:7.3f}")
