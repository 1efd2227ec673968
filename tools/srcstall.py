"""Profiling aid: stall samples per CUDA source line from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows, fname = [], ""
for r in csv.reader(open(path)):
    if len(r) == 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if len(r) > 8 and r[0] and r[0] != "Line No" and r[0].isdigit():
        num = lambda x: int(x) if x.strip().isdigit() else 0
        rows.append((num(r[4]), num(r[7]), f"{fname}:{r[0]}", r[1].strip()[:90]))
tot = sum(x[0] for x in rows) or 1
for s, i, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}%  inst {i:>10d}  {loc:>18}  {src}")
