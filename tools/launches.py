"""Profiling aid: per-kernel mean duration (us) from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys

d = collections.defaultdict(list)
for r in csv.DictReader(l for l in open(sys.argv[1]) if not l.startswith("==")):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        d[r["Kernel Name"].split("(")[0].split("::")[-1][:40]].append(v / (1000.0 if r["Metric Unit"] == "nsecond" else 1.0))
tot = 0.0
for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1]) / len(kv[1])):
    print(f"{k:42s} n={len(v):3d} mean={sum(v) / len(v):8.1f} us")
