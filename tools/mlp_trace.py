"""Profiling aid: per-layer event timeline of the TS-mode MLP (k_mlp_ts) from a
build with -DNVC_MLP_TRACE (clock64 stamps of CTA 0's first 8 tiles per
warpgroup).  Builds libnvc_trace.so if needed, runs the C2 query front on
2,073,600 random points and prints, per layer, the mean cycles from MMA issue
to commit, commit to epilogue wake-up, the epilogue, and the epilogue's end to
the next layer's MMA issue.  Usage: mlp_trace.py"""
import ctypes
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_05930_b200 import _lib, build  # noqa: E402

extra = sys.argv[1:]          # e.g. -DNVC_MLP_NOSTORE (experiments)
so = os.path.join(ROOT, "paper_2506_05930_b200", "libnvc_trace" + "".join(e.lower().replace("-d", "_") for e in extra) + ".so")
build.build(defs=["-DNVC_MLP_TRACE"] + extra, out=so)
_lib._lib = _lib.load(so)
import torch  # noqa: E402

from paper_2506_05930_b200 import MODE_LIGHTS, HashGridConfig, VisibilityCache  # noqa: E402

lo, hi = np.array([-3.0, 0.0, -2.2]), np.array([3.0, 1.5, 3.0])
c = VisibilityCache(MODE_LIGHTS, 32, HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2,
                                                    aabb_min=lo, aabb_max=hi), hidden_dims=(64, 64, 64))
P = 1920 * 1080
pos = torch.from_numpy(np.random.default_rng(0).uniform(lo, hi, (P, 3))).cuda()
ws = c.query_workspace(P)
for _ in range(3):
    _lib.call("nvc_query_front", c.model, pos.data_ptr(), P, _lib.ptr(ws), _lib.stream_ptr())
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10):
    _lib.call("nvc_query_front", c.model, pos.data_ptr(), P, _lib.ptr(ws), _lib.stream_ptr())
e1.record()
torch.cuda.synchronize()
print(f"query front (encoder + MLP): {e0.elapsed_time(e1) / 10 * 1000:.1f} us")
tr = np.zeros((4, 8, 4, 6), dtype=np.int64)
_lib._lib.nvc_mlp_trace_get.argtypes = [ctypes.c_void_p]
assert _lib._lib.nvc_mlp_trace_get(tr.ctypes.data) == 0
t0 = tr[tr > 0].min()
t = (tr - t0).astype(np.float64)
names = ["issue->commit", "commit->wake", "epilogue", "done->next issue"]
for layer in range(4):
    iss, com, wake, done = (t[:, 1:7, layer, e] for e in range(4))   # tiles 1-6 (steady state)
    nxt = t[:, 1:7, layer + 1, 0] if layer < 3 else t[:, 2:8, 0, 0]
    row = [(com - iss).mean(), (wake - com).mean(), (done - wake).mean(), (nxt - done).mean()]
    print(f"layer {layer}: " + "  ".join(f"{n} {v:7.0f}" for n, v in zip(names, row)))
per_tile = (t[:, 7, 0, 0] - t[:, 1, 0, 0]) / 6
print("cycles per tile per warpgroup:", " ".join(f"{x:.0f}" for x in per_tile))
a0 = (t[:, 2:8, 0, 0] - t[:, 2:8, 0, 4]).mean()
tail = (t[:, 1:7, 3, 5] - t[:, 1:7, 3, 3]).mean()
wake_after_tail = (t[:, 2:8, 0, 2] - t[:, 1:7, 3, 5]).mean()
prev_done_to_a0 = (t[:, 2:8, 0, 4] - t[:, 1:7, 3, 3]).mean()
print(f"output tail (sigmoid + stores) {tail:.0f}; next layer-0 wake after the tail {wake_after_tail:.0f}; "
      f"prev output done -> a0 ready {prev_done_to_a0:.0f}; a0 ready -> layer-0 issue {a0:.0f}")
print("warpgroup 0, tile 3 stamps (issue, commit, wake, done, a0, tail) per layer:")
print((t[0, 3] - t[0, 3, 0, 0]).astype(int))
