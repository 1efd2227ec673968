"""Diagnostic (CPU): how many triangles reach the per-lane culling loop of the
warp-cooperative any-hit (geometry.cu any_hit_bf_warp) for the C2 training
batch's shadow rays, under
  leaf-union: a triangle's BVH leaf box against the union of the warp's
              segment boxes (the current warp filter), and
  shaft:      the triangle's box (leaf box for unboxed slivers) against the
              hull of the warp's origin box and end box (the swept box
              (1-s) A + s B, s in [0, 1]: an exact box-vs-hull test),
plus the per-lane survivors of the plane + crossing-box filters.
Warps = 32 Morton-bucketed rows x one light, as k_targets_sorted.
Usage: shaft_sim.py [n_frames] [boxes32|rooms128]"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import vc_oracle as O  # noqa: E402
from paper_2506_05930_b200 import scene_from_dict  # noqa: E402
from paper_2506_05930_b200.scene import PLANE_MARGIN, shadow_accel, shadow_epsilon  # noqa: E402
from paper_2506_05930_b200.scenes import boxes_scene, rooms_scene  # noqa: E402

s = scene_from_dict(rooms_scene(128) if len(sys.argv) > 2 and sys.argv[2] == "rooms128" else boxes_scene(32))
c = s.camera
sa = O.SceneArrays(s.triangles_v0, s.triangles_v1, s.triangles_v2, s.tri_material, s.tri_light, s.lt_kind,
                   s.lt_verts, s.lt_normal, s.lt_radiance, s.mat_albedo,
                   np.concatenate([c.position, c.look_at, c.up, [c.fov_deg, c.width, c.height]]))
b = s.bvh
plane, box, leaf, parent, R = shadow_accel(b)
eps = shadow_epsilon(b)
ntri = b.v0.shape[0]
leaf_lo = b.node_min[leaf].astype(np.float32)
leaf_hi = b.node_max[leaf].astype(np.float32)
boxed = box[:ntri, 3] == 0.0
f_lo = np.where(boxed[:, None], box[:ntri, 0:3], leaf_lo)
f_hi = np.where(boxed[:, None], box[:ntri, 4:7], leaf_hi)


def morton(pos):
    lo, hi = s.aabb_min, s.aabb_max
    q = np.clip(((pos - lo) / (hi - lo) * 16).astype(np.int64), 0, 15)
    code = np.zeros(len(pos), np.int64)
    for bit in range(4):
        for a in range(3):
            code |= ((q[:, a] >> bit) & 1) << (3 * bit + a)
    return np.argsort(code, kind="stable")


def shaft_keep(A_lo, A_hi, B_lo, B_hi, t_lo, t_hi):
    """exists s in [0,1]: box (1-s)A + sB overlaps t (per triangle rows)."""
    s_lo, s_hi = np.zeros(len(t_lo)), np.ones(len(t_lo))
    for a in range(3):
        for (p0, d, bound, le) in ((A_lo[a], B_lo[a] - A_lo[a], t_hi[:, a], True),
                                   (A_hi[a], B_hi[a] - A_hi[a], t_lo[:, a], False)):
            # le: p0 + s d <= bound ; else p0 + s d >= bound
            if d == 0.0:
                ok = (p0 <= bound) if le else (p0 >= bound)
                s_hi = np.where(ok, s_hi, -1.0)
                continue
            t = (bound - p0) / d
            if (d > 0) == le:
                s_hi = np.minimum(s_hi, t)
            else:
                s_lo = np.maximum(s_lo, t)
    return s_lo <= s_hi


nfr = int(sys.argv[1]) if len(sys.argv) > 1 else 1
stats = {"leaf_union": [], "shaft": [], "shaft_leafbox": [], "shaft_guarded": [], "shaft_guarded+plane": [], "lane_cull": []}
nrm = plane[:ntri, :3].astype(np.float64)
boxable = boxed & (np.abs(nrm).sum(1) > 0)
for fr in range(nfr):
    key = (0, fr, 0)
    world = O.world_samples(sa, 4096, O.Stream(*key, "world-samples"))
    screen = O.screen_samples(sa, 4096, O.Stream(*key, "screen-samples"))
    pos = np.concatenate([world, screen])
    order = morton(pos)
    rng = np.random.default_rng(fr)
    for j in range(sa.k):
        y = sa.light_points(np.full(len(pos), j), rng.random((len(pos), 2)))
        for w0 in range(0, len(pos), 32):
            idx = order[w0:w0 + 32]
            o, yy = pos[idx], y[idx]
            dd = yy - o
            dist = np.linalg.norm(dd, axis=1)
            d = dd / dist[:, None]
            tmax = np.maximum(dist - eps, eps + 1e-12)
            p0 = (o + eps * d).astype(np.float32)
            p1 = (o + tmax[:, None] * d).astype(np.float32)
            m = (PLANE_MARGIN * ((R + np.abs(p0).max(1)) + np.abs(p1).max(1)) + 1e-30).astype(np.float32)
            of = o.astype(np.float32)
            # current: leaf box vs union of [min(o, p1) - m, max(o, p1) + m]
            ulo = (np.minimum(of, p1) - m[:, None]).min(0)
            uhi = (np.maximum(of, p1) + m[:, None]).max(0)
            cand = np.all((leaf_lo <= uhi) & (leaf_hi >= ulo), axis=1)
            stats["leaf_union"].append(cand.sum())
            A_lo = (np.minimum(of, p0) - m[:, None]).min(0)
            A_hi = (np.maximum(of, p0) + m[:, None]).max(0)
            B_lo, B_hi = (p1 - m[:, None]).min(0), (p1 + m[:, None]).max(0)
            stats["shaft"].append(shaft_keep(A_lo, A_hi, B_lo, B_hi, f_lo, f_hi).sum())
            k_leaf = shaft_keep(A_lo, A_hi, B_lo, B_hi, leaf_lo, leaf_hi)
            stats["shaft_leafbox"].append(k_leaf.sum())
            # tri-box culling only where every lane's segment crosses the plane at
            # |s1 - s0| > 4 m: the gap between A's and B's projections onto the normal
            ca, ra = (A_lo + A_hi) / 2, (A_hi - A_lo) / 2
            cb, rb = (B_lo + B_hi) / 2, (B_hi - B_lo) / 2
            pa, pb = nrm @ ca, nrm @ cb
            ea, eb = np.abs(nrm) @ ra, np.abs(nrm) @ rb
            gap = np.abs(pb - pa) - ea - eb
            ok = boxable & (gap > 4.5 * m.max())
            k_tri = shaft_keep(A_lo, A_hi, B_lo, B_hi, f_lo, f_hi)
            stats["shaft_guarded"].append((k_leaf & (~ok | k_tri)).sum())
            off = plane[:ntri, 3].astype(np.float64)
            lo_s = np.minimum(pa - ea, pb - eb) - off
            hi_s = np.maximum(pa + ea, pb + eb) - off
            side = (lo_s > m.max()) | (hi_s < -m.max())
            stats["shaft_guarded+plane"].append((k_leaf & (~ok | k_tri) & ~(side & (np.abs(nrm).sum(1) > 0))).sum())
            # per-lane plane filter survivors (union over lanes) among all triangles
            s0 = p0 @ plane[:ntri, :3].T - plane[:ntri, 3]
            s1 = p1 @ plane[:ntri, :3].T - plane[:ntri, 3]
            keep = ~((np.minimum(s0, s1) > m[:, None]) | (np.maximum(s0, s1) < -m[:, None]))
            stats["lane_cull"].append(keep.any(0).sum())
for k, v in stats.items():
    v = np.array(v)
    print(f"{k:>20}: mean {v.mean():6.2f} triangles per warp (of {ntri}), p50 {np.median(v):.0f}, p90 {np.percentile(v, 90):.0f}")
