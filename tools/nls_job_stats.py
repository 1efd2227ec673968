"""Diagnostic: per-warp imbalance of NLS Philox jobs (4-light groups with a nonzero lum + the light-point pair)."""
import sys, torch, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2506_05930_b200.scene import scene_from_dict
from paper_2506_05930_b200.scenes import boxes_scene, rooms_scene
from paper_2506_05930_b200.render import gbuffer_device
from paper_2506_05930_b200.sampling import PixelCtx
for name, sc in (("boxes32", boxes_scene(32)), ("rooms128", rooms_scene(128))):
    scene = scene_from_dict(sc)
    cam = scene.camera.resized(1920, 1080)
    P = 1920 * 1080
    pos, nrm, alb, hit, _ = gbuffer_device(scene, cam, 0, P)
    ctx = PixelCtx(scene, pos, nrm, alb)
    m = ctx.mask_device().cpu().numpy().view(np.uint32)
    K = scene.n_lights if hasattr(scene, 'n_lights') else len(scene.lights)
    W = (K + 31) // 32
    m = m.reshape(W, P)
    jobs = np.ones(P, np.int64)
    for w in range(W):
        for g in range(8):
            jobs += ((m[w] >> (4 * g)) & 15) != 0
    warp = jobs.reshape(-1, 32)
    print(name, "mean jobs/pixel", jobs.mean(), "warp max mean", warp.max(1).mean(),
          "balanced ceil", np.ceil(warp.sum(1) / 32).mean(), "ratio", warp.max(1).mean() / np.ceil(warp.sum(1) / 32).mean())

if "--reverse" not in sys.argv:
    sys.exit(0)
# Reverse-scan estimate: the WRS selection is the LAST light with u*s_k < w_k, so a
# scan from the top group down could stop at the selected light's group.  Blocks a
# reverse scan would need = nonzero groups at or above the selected group (+1 pair).
from paper_2506_05930_b200 import MODE_LIGHTS, HashGridConfig, TrainFrameConfig, VisibilityCache
from paper_2506_05930_b200 import rng as R
from paper_2506_05930_b200.sampling import nls_sample_device
from paper_2506_05930_b200.training import train_frame_device
scene = scene_from_dict(boxes_scene(32))
cam = scene.camera.resized(1920, 1080)
P = 1920 * 1080
pos, nrm, alb, hit, _ = gbuffer_device(scene, cam, 0, P)
ctx = PixelCtx(scene, pos, nrm, alb)
m = ctx.mask_device().cpu().numpy().view(np.uint32)
grp = np.stack([((m >> (4 * g)) & 15) != 0 for g in range(8)], 1)       # (P, 8)
grid = HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2, aabb_min=scene.aabb_min,
                      aabb_max=scene.aabb_max)
cache = VisibilityCache(MODE_LIGHTS, 32, grid, seed=0, hidden_dims=(64, 64, 64), device=torch.device("cuda", 0))
cfg = TrainFrameConfig(n_world=4096, n_screen=4096, seed=0)
for frames in (0, 60):
    for f in range(frames):
        train_frame_device(scene, cam, cache, cfg, frame=f)
    ids, _, _ = nls_sample_device(ctx, cache, R.stream_key(0, 7, "light-select"), 0)
    ids = ids.cpu().numpy()
    gs = np.where(ids >= 0, ids // 4, 0)
    need = np.array([grp[p, gs[p]:].sum() for p in range(0, P, 97)]) + 1
    fwd = grp[::97].sum(1) + 1
    warp_need = need[: (need.size // 32) * 32].reshape(-1, 32)
    print(f"after {frames} frames: forward blocks/pixel {fwd.mean():.3f}  reverse mean {need.mean():.3f}"
          f"  (sampled pixels; a lane-per-pixel warp pays ~max over lanes)")
