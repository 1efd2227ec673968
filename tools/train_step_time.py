"""Diagnostic: device time of one C2-shaped training step (accumulate_grads on
an 8192-row batch: encode, MLP fwd+bwd, scatter, reduce) for the fp32 SIMT
step and the tcgen05 step (NVC_TRAIN_TC=1).  Usage: train_step_time.py [iters] [tc|simt|both]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2506_05930_b200 import MODE_LIGHTS, HashGridConfig, VisibilityCache, scene_from_dict  # noqa: E402
from paper_2506_05930_b200.scenes import boxes_scene  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 50
which = sys.argv[2] if len(sys.argv) > 2 else "both"
s = scene_from_dict(boxes_scene(32))
rng = np.random.default_rng(0)
pos = torch.from_numpy(rng.uniform(s.aabb_min, s.aabb_max, (8192, 3))).cuda()
tgt = torch.from_numpy((rng.random((8192, 32)) < 0.5).astype(np.float32)).cuda()
c = VisibilityCache(MODE_LIGHTS, 32, HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2,
                                                    aabb_min=s.aabb_min, aabb_max=s.aabb_max),
                    seed=0, hidden_dims=(64, 64, 64))
for tc in ([False, True] if which == "both" else [which == "tc"]):
    if tc:
        os.environ["NVC_TRAIN_TC"] = "1"
    else:
        os.environ.pop("NVC_TRAIN_TC", None)
    for _ in range(5):
        c.accumulate_grads(pos, tgt)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        c.accumulate_grads(pos, tgt)
    e1.record()
    torch.cuda.synchronize()
    print(f"{'tc' if tc else 'simt'}: {1000 * e0.elapsed_time(e1) / iters:.1f} us per accumulate_grads")
