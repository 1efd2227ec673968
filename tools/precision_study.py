"""Diagnostic: how the C2 60-frame loss curve depends on the training GEMMs'
operand precision.  The fp32 SIMT step rounds every GEMM operand (weights,
activations, deltas) to m significant bits (NVC_T3_BITS=m) -- the ideal of a
split-operand tensor-core step with m-bit pieces -- and the curve is compared
with the reference's f32 / f64 runs (tests/golden/curves.npz).  Also runs the
tensor-core step (NVC_TRAIN_TC=1) for comparison.
Usage: precision_study.py [m ...]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2506_05930_b200 import (MODE_LIGHTS, HashGridConfig, TrainFrameConfig, VisibilityCache,  # noqa: E402
                                   scene_from_dict, train_frame)
from paper_2506_05930_b200.scenes import boxes_scene  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", "curves.npz"))
ref32, ref64 = g["c2_loss60_f32"], g["c2_loss60_f64"]
scene = scene_from_dict(boxes_scene(32))


def curve():
    c = VisibilityCache(MODE_LIGHTS, 32, HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2,
                                                        aabb_min=scene.aabb_min, aabb_max=scene.aabb_max),
                        seed=0, hidden_dims=(64, 64, 64))
    return np.array([train_frame(scene, scene.camera, c, TrainFrameConfig(), frame=f) for f in range(60)])


def report(tag, got):
    r32, r64 = np.abs(got - ref32) / ref32, np.abs(got - ref64) / ref64
    print(f"{tag:>10}: max rel vs ref f32 {r32.max():.2e} (mean {r32.mean():.2e}), vs f64 {r64.max():.2e} "
          f"(mean {r64.mean():.2e}); first frame > 1e-2: {int(np.argmax(r32 > 1e-2)) if (r32 > 1e-2).any() else '-'}; "
          f"frames 40-59 mean loss {got[40:].mean():.5f} (ref f32 {ref32[40:].mean():.5f}, "
          f"{got[40:].mean() / ref32[40:].mean() - 1:+.2%})", flush=True)


spread = np.abs(ref32 - ref64) / ref64
print(f"reference f32 vs f64 spread: max {spread.max():.2e} mean {spread.mean():.2e}")
bits = [int(b) for b in sys.argv[1:]] or [0, 23, 22, 21, 20, 18, 16]
for m in bits:
    os.environ.pop("NVC_TRAIN_TC", None)
    if m:
        os.environ["NVC_T3_BITS"] = str(m)
    else:
        os.environ.pop("NVC_T3_BITS", None)
    report(f"fp32" if not m else f"{m} bits", curve())
for m, what, name in ((23, 1, "weights"), (23, 2, "activations"), (23, 4, "deltas"),
                      (17, 6, "act+delta"), (16, 6, "act+delta"), (14, 6, "act+delta")):
    os.environ["NVC_T3_BITS"], os.environ["NVC_T3_WHAT"] = str(m), str(what)
    report(f"{m}b {name}", curve())
os.environ.pop("NVC_T3_BITS", None)
os.environ.pop("NVC_T3_WHAT", None)
os.environ["NVC_TRAIN_TC"] = "1"
report("tcgen05", curve())
