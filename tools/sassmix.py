"""Profiling aid: per-opcode instruction mix from an `ncu --page source --csv --print-source sass` export."""
import collections
import csv
import sys

path, pixels = sys.argv[1], float(sys.argv[2])
ops, stalls = collections.Counter(), collections.Counter()
hdr, tot = None, 0
for r in csv.reader(open(path)):
    if r and r[0] == "Address":
        hdr = r
        ie, src, st = hdr.index("Instructions Executed"), hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
        continue
    if hdr is None or len(r) <= ie or not r[ie].strip().isdigit():
        continue
    n = int(r[ie])
    tot += n
    toks = r[src].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
    ops[op] += n
    stalls[op] += int(r[st] or 0)
print("total warp inst", tot, "per unit", tot * 32 / pixels)
for op, n in ops.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 45):
    print(f"{op:28s} {n * 32 / pixels:8.1f}/unit  stall {stalls[op]}")
