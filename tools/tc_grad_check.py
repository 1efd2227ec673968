"""Diagnostic: tcgen05 training-step gradients (NVC_TRAIN_TC=1) against the fp32 SIMT step, per parameter block."""
import os, sys, numpy as np, torch
sys.path.insert(0, '/root/repo')
from paper_2506_05930_b200 import MODE_LIGHTS, HashGridConfig, VisibilityCache, scene_from_dict, TrainFrameConfig, train_frame
from paper_2506_05930_b200.scenes import boxes_scene, boxes_point_scene
sys.path.insert(0, '/root/repo/tests')
from conftest import golden
g = golden("training")
def grads(scene, levels, tsize, hidden, k, pos, tgt, tc):
    if tc: os.environ["NVC_TRAIN_TC"] = "1"
    else: os.environ.pop("NVC_TRAIN_TC", None)
    c = VisibilityCache(MODE_LIGHTS, k, HashGridConfig(levels=levels, table_size=tsize, features_per_level=2, aabb_min=scene.aabb_min, aabb_max=scene.aabb_max), seed=0, hidden_dims=hidden)
    c.set_compact(False)
    p = torch.from_numpy(pos).cuda(); t = torch.from_numpy(tgt.astype(np.float32)).cuda()
    loss = c.accumulate_grads(p, t)
    torch.cuda.synchronize()
    return c.grad_fx.double().cpu().numpy() * 2.0**-48, loss.cpu().numpy(), c
s8 = scene_from_dict(boxes_point_scene(8))
a, la, c = grads(s8, 8, 1<<14, (64,64), 8, g["c1_pos"], g["c1_tgt"], False)
b, lb, _ = grads(s8, 8, 1<<14, (64,64), 8, g["c1_pos"], g["c1_tgt"], True)
n = c.grid_cfg.param_count
print("C1 loss", la, lb)
for name, sl in (("grid", slice(0, n)), ("mlp", slice(n, None))):
    x, y = a[sl], b[sl]
    print(name, "max|d|", np.abs(x-y).max(), "max|x|", np.abs(x).max(), "rel", np.abs(x-y).max()/np.abs(x).max())
s32 = scene_from_dict(boxes_scene(32))
a, la, c = grads(s32, 16, 1<<19, (64,64,64), 32, g["b32_pos"], g["b32_tgt"], False)
b, lb, _ = grads(s32, 16, 1<<19, (64,64,64), 32, g["b32_pos"], g["b32_tgt"], True)
n = c.grid_cfg.param_count
print("C2 loss", la, lb)
for name, sl in (("grid", slice(0, n)), ("mlp", slice(n, None))):
    x, y = a[sl], b[sl]
    print(name, "max|d|", np.abs(x-y).max(), "max|x|", np.abs(x).max(), "rel", np.abs(x-y).max()/np.abs(x).max())

# per-parameter-block relative errors (C2)
offs = c._layer_offs
dims = c.net_cfg.layer_dims
for i, ((wo, bo), (fo, fi)) in enumerate(zip(offs, dims)):
    for nm, sl in ((f"w{i}", slice(wo, wo + fo * fi)), (f"b{i}", slice(bo, bo + fo))):
        x, y = a[sl], b[sl]
        print(nm, "max|x|", f"{np.abs(x).max():.3e}", "max|d|/max|x|", f"{np.abs(x-y).max()/np.abs(x).max():.3e}",
              "median rel", f"{np.median(np.abs(x-y)/np.maximum(np.abs(x),1e-30)):.3e}")
x, y = a[:n], b[:n]
nz = np.abs(x) > 1e-3 * np.abs(x).max()
print("grid: rel err percentiles (|x| > 1e-3 max):", np.percentile(np.abs(x[nz]-y[nz])/np.abs(x[nz]), [50, 90, 99, 100]))
