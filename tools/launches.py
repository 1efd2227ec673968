"""Profiling aid: per-kernel mean duration and DRAM bytes from an
`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv` launch list."""
import collections
import csv
import json
import sys


def load(path):
    d = collections.defaultdict(lambda: collections.defaultdict(list))
    for r in csv.DictReader(l for l in open(path) if not l.startswith("==")):
        name = r["Kernel Name"].split("(")[0].split("::")[-1].strip()
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        if r["Metric Name"] == "gpu__time_duration.sum":
            v = v / 1000.0 if unit in ("ns", "nsecond") else (v * 1000.0 if unit in ("ms", "msecond") else v)   # -> us
        d[name][r["Metric Name"]].append(v)
    return d


if __name__ == "__main__":
    d = load(sys.argv[1])
    rows = []
    for k, m in d.items():
        t = m.get("gpu__time_duration.sum", [])
        if not t:
            continue
        rd, wr = m.get("dram__bytes_read.sum", []), m.get("dram__bytes_write.sum", [])
        rows.append((sum(t) / len(t), k, len(t), (sum(rd) / len(rd)) if rd else None, (sum(wr) / len(wr)) if wr else None))
    rows.sort(reverse=True)
    for us, k, n, rd, wr in rows:
        dram = (f"  dram r {rd / 1e6:8.1f} MB" + (f"  w {wr / 1e6:8.1f} MB" if wr is not None else "")) if rd is not None else ""
        print(f"{k:32s} n={n:3d} mean={us:9.1f} us{dram}")
    if len(sys.argv) > 2:   # write {kernel: dram bytes per launch} for bench.py's roofline.traffic
        out = {k: int(rd + (wr or 0)) for us, k, n, rd, wr in rows if rd is not None}
        json.dump(out, open(sys.argv[2], "w"), indent=1, sort_keys=True)
