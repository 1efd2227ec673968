"""Diagnostic: per-frame kernel timeline from a CUPTI trace (bench.py with
NVC_TIMELINE=<trace.json>): each kernel's stream, start offset in its frame and
duration, and the overlap of the query and training chains.
Usage: timeline.py trace.json [frame_anchor_kernel]"""
import json
import sys
from collections import defaultdict

ev = json.load(open(sys.argv[1]))
ev = ev["traceEvents"] if isinstance(ev, dict) else ev
ks = sorted((e for e in ev if e.get("cat") == "kernel"), key=lambda e: e["ts"])
anchor = sys.argv[2] if len(sys.argv) > 2 else "k_enc_tiles2"
import re  # noqa: E402


def short(n):
    m = re.search(r"(k_\w+)(<[^(]*?>)?\(", n)
    return (m.group(1) + (m.group(2) or "")) if m else n[:40]
starts = [e["ts"] for e in ks if anchor in e["name"]]
print(f"{len(ks)} kernels, {len(starts)} frames (anchor {anchor})")
if len(starts) > 2:
    per = [b - a for a, b in zip(starts, starts[1:])]
    print("frame period (anchor to anchor) us:", " ".join(f"{x:.0f}" for x in per))
# one steady frame in detail: the window [starts[-3], starts[-2])
if len(starts) >= 3:
    t0, t1 = starts[-3], starts[-2]
    print(f"\nframe window {t1 - t0:.1f} us:")
    print(f"{'kernel':40s} {'stream':>6s} {'start':>7s} {'end':>7s} {'dur':>6s}")
    for e in ks:
        s, d = e["ts"], e["dur"]
        if s + d > t0 and s < t1:
            print(f"{short(e['name']):40s} {e['args'].get('stream', '?'):>6} {s - t0:7.1f} {s + d - t0:7.1f} {d:6.1f}")
# busy fraction: union of kernel intervals over the steady frames
iv = sorted((e["ts"], e["ts"] + e["dur"]) for e in ks if starts and starts[1] <= e["ts"] < starts[-1])
busy, cur = 0.0, None
for a, b in iv:
    if cur is None or a > cur[1]:
        if cur:
            busy += cur[1] - cur[0]
        cur = [a, b]
    else:
        cur[1] = max(cur[1], b)
if cur:
    busy += cur[1] - cur[0]
if len(starts) > 2:
    span = starts[-1] - starts[1]
    print(f"\nGPU busy (any kernel running) {busy / span:.1%} of {span:.0f} us")
tot = defaultdict(float)
for e in ks:
    if starts and starts[1] <= e["ts"] < starts[-1]:
        tot[short(e["name"])] += e["dur"]
n = max(len(starts) - 2, 1)
print("\nper-frame kernel time (us):")
for k, v in sorted(tot.items(), key=lambda t: -t[1]):
    print(f"  {k:40s} {v / n:7.1f}")
print(f"  {'sum':40s} {sum(tot.values()) / n:7.1f}")
