"""Profiling aid: event timeline of k_mlp_wg (CTA 0) from the NVC_TRACE build.

    python -m paper_2506_05930_b200.build --trace && python tools/trace_mlp.py
"""
import collections
import ctypes
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_05930_b200 import MODE_LIGHTS, HashGridConfig, VisibilityCache, _lib  # noqa: E402
from paper_2506_05930_b200 import rng as R  # noqa: E402
from paper_2506_05930_b200.render import gbuffer_device  # noqa: E402
from paper_2506_05930_b200.sampling import PixelCtx, nls_sample_device  # noqa: E402
from paper_2506_05930_b200.scene import scene_from_dict  # noqa: E402
from paper_2506_05930_b200.scenes import boxes_scene  # noqa: E402

lib = _lib.load(os.path.join(os.path.dirname(_lib.LIB_PATH), "libnvc_trace.so"))
_lib._lib = lib
lib.nvc_wg_trace.restype = ctypes.c_int
lib.nvc_wg_trace.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
scene = scene_from_dict(boxes_scene(32))
cam = scene.camera.resized(1920, 1080)
pos, nrm, alb, _, _ = gbuffer_device(scene, cam)
ctx = PixelCtx(scene, pos, nrm, alb)
ctx.lum_device()
grid = HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2, aabb_min=scene.aabb_min,
                      aabb_max=scene.aabb_max)
cache = VisibilityCache(MODE_LIGHTS, 32, grid, hidden_dims=(64, 64, 64))
for i in range(3):
    nls_sample_device(ctx, cache, R.stream_key(0, i, "light-select"))
torch.cuda.synchronize()
lib.nvc_wg_trace(None, 0, 1)
nls_sample_device(ctx, cache, R.stream_key(0, 9, "light-select"))
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 32768)()
n = lib.nvc_wg_trace(ctypes.addressof(buf), 32768, 0)
raw = [int(buf[g * 4096 + i]) for g in range(8) for i in range(n) if int(buf[g * 4096 + i])]
ev = sorted((b >> 16, (b >> 12) & 15, (b >> 8) & 15, (b >> 4) & 15, b & 15) for b in raw)
t0 = ev[0][0]
last = {}
dur = collections.defaultdict(list)
names = {(1, 2): "wait acc", (2, 3): "epilogue", (3, 4): "handoff", (4, 5): "issue", (5, 6): "x", (6, 7): "mma0",
         (7, 8): "mma1-3", (8, 9): "commit"}
for t, g, c, l, s in ev:
    key = (g, l, s)
    if c in (2, 3, 4, 7, 8, 9) and (key, c - 1) in last:
        dur[(names[(c - 1, c)], "out" if l == 3 else "hid")].append(t - last[(key, c - 1)])
    if c == 6 and (key, 4) in last:
        dur[("issue->mma", "out" if l == 3 else "hid")].append(t - last[(key, 4)])
    if c == 5 and (key, 4) in last:
        dur[("issue", "out" if l == 3 else "hid")].append(t - last[(key, 4)])
    last[(key, c)] = t
print(n, "events; span", ev[-1][0] - t0, "cycles")
for k, v in sorted(dur.items()):
    print(f"{k[0]:10s} {k[1]}: n={len(v):5d} median={statistics.median(v):8.0f} mean={statistics.mean(v):8.0f} "
          f"p90={sorted(v)[int(0.9 * len(v))]:8.0f}")
with open(os.path.join("gpurun_out", "trace_mlp.txt"), "w") as fh:
    for t, g, c, l, s in ev[:3000]:
        fh.write(f"{t - t0:9d} wg{g} c{c} l{l} s{s}\n")
