"""Diagnostic: distinct 32-B sectors per warp-wide x-pair gather, per hash-grid level, for
row-major (32x1) and 2-D (8x4, 16x2) pixel-to-lane mappings over a 256x128 window of the C2
1080p G-buffer (oracle geometry on the CPU).  Result: profiles/r2_gather_sectors.txt."""
import sys, numpy as np
sys.path.insert(0, '/root/repo')
from oracle import vc_oracle as O
from paper_2506_05930_b200.scene import scene_from_dict
from paper_2506_05930_b200.scenes import boxes_scene
s = scene_from_dict(boxes_scene(32))
W, H = 1920, 1080
cam = np.array([*s.camera.position, *s.camera.look_at, *s.camera.up, s.camera.fov_deg, W, H], float)
sa = O.SceneArrays(s.triangles_v0, s.triangles_v1, s.triangles_v2, s.tri_material, s.tri_light, s.lt_kind,
                   s.lt_verts, s.lt_normal, s.lt_radiance, s.mat_albedo, cam)
# a 256x128 window in the image center, 2 mappings
x0, y0, w, h = 832, 476, 256, 128
ys, xs = np.mgrid[y0:y0+h, x0:x0+w]
pix = (ys * W + xs).reshape(-1)
jit = O.uniform_at(O.stream_key("primary"), np.stack([2 * pix, 2 * pix + 1], 1))
o, d = sa.camera_rays(xs.reshape(-1) + jit[:, 0], ys.reshape(-1) + jit[:, 1])
gb = sa.trace(o, d)
pos = gb["position"].reshape(h, w, 3)
g = O.Grid(levels=16, features_per_level=2, table_size=1 << 19, aabb_min=s.aabb_min, aabb_max=s.aabb_max)
def warps_rowmajor():
    return [pos[r, c:c+32].reshape(-1, 3) for r in range(h) for c in range(0, w, 32)]
def warps_block(bw, bh):
    return [pos[r:r+bh, c:c+bw].reshape(-1, 3) for r in range(0, h, bh) for c in range(0, w, bw)]
for name, ws in (("32x1", warps_rowmajor()), ("8x4", warps_block(8, 4)), ("16x2", warps_block(16, 2))):
    tot = 0
    per_level = []
    allp = np.concatenate(ws)
    q = O.normalize(g, allp)
    for l in range(16):
        idx, _ = O.level_lookup(g, l, q)      # (n, 8) int64; x-pair slot = corner with bx=0 -> corners 0..3
        slots = idx[:, :4]                      # x-pair: the bx=0 corners carry both x-neighbours
        sec = slots // 4                        # 8-B slots, 32-B sectors
        n = 0
        for wi in range(len(ws)):
            ss = sec[wi*32:(wi+1)*32]
            n += sum(len(np.unique(ss[:, c])) for c in range(4))
        per_level.append(n / len(ws) / 4)
        tot += n
    print(name, "sectors/request per level:", " ".join(f"{x:.1f}" for x in per_level), "| mean", round(np.mean(per_level), 2))
