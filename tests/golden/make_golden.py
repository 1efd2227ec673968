"""Generate the golden fixtures by running the REFERENCE `viscache` package.

Run once in the build container (the only place /root/reference exists):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports the reference read-only, evaluates it on small seeded inputs, and
writes compressed .npz files next to this script.  Nothing at run time (tests,
smoke, bench) reads /root/reference; the fixtures are the portable record of
what the reference computes.  Inputs that are large but cheap to regenerate
(feature tables, He weights) are regenerated in the tests from the same numpy
Philox streams and pinned here by checksum.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

from viscache import rng as R  # noqa: E402  (reference, read-only)
from viscache.cache import MODE_LIGHTS, VisibilityCache  # noqa: E402
from viscache.geometry import visibility_batch  # noqa: E402
from viscache.hashgrid import (HashGridConfig, _level_lookup, _normalize,  # noqa: E402
                               encode_batch, grad_from_ctx, init_params)
from viscache.mlp import (AdamState, MLPConfig, adam_step, backward_l2,  # noqa: E402
                          forward, he_init, l2_loss)
from viscache.render import make_gbuffer, shade_batch  # noqa: E402
from viscache.sampling import (PixelCtx, neural_di_batch, nls_sample_batch,  # noqa: E402
                               wrs_select_batch)
from viscache.scene import Camera, scene_from_dict  # noqa: E402
from viscache.scenes import boxes_scene, rooms_scene  # noqa: E402
from viscache.training import (TrainFrameConfig, compute_visibility_targets,  # noqa: E402
                               gen_screen_samples, gen_world_samples, train_frame)


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def point_light_dict(n: int) -> dict:
    """C1 fixture: boxes_scene(n) with every rect light replaced by a point
    light at its centroid carrying intensity = radiance * area."""
    d = boxes_scene(n)
    lights = []
    for lt in d["lights"]:
        c = np.array(lt["corner"], float)
        u = np.array(lt["edge_u"], float)
        v = np.array(lt["edge_v"], float)
        area = float(np.linalg.norm(np.cross(u, v)))
        lights.append({"type": "point", "position": list(c + 0.5 * u + 0.5 * v),
                       "intensity": [area * r for r in lt["radiance"]]})
    d["lights"] = lights
    d["camera"] = dict(d["camera"], width=64, height=64)
    return d


def scene_arrays(prefix: str, s, out: dict) -> None:
    out[prefix + "v0"] = s.triangles_v0
    out[prefix + "v1"] = s.triangles_v1
    out[prefix + "v2"] = s.triangles_v2
    out[prefix + "tri_material"] = s.tri_material
    out[prefix + "tri_light"] = s.tri_light
    out[prefix + "lt_kind"] = s.lt_kind
    out[prefix + "lt_verts"] = s.lt_verts
    out[prefix + "lt_normal"] = s.lt_normal
    out[prefix + "lt_area"] = s.lt_area
    out[prefix + "lt_radiance"] = s.lt_radiance
    out[prefix + "mat_albedo"] = s.mat_albedo
    out[prefix + "aabb_min"] = s.aabb_min
    out[prefix + "aabb_max"] = s.aabb_max
    b = s.bvh
    for k in ("node_min", "node_max", "node_left", "node_right", "node_start",
              "node_count", "perm"):
        out[prefix + "bvh_" + k] = getattr(b, k)
    c = s.camera
    out[prefix + "cam"] = np.array([*c.position, *c.look_at, *c.up, c.fov_deg,
                                    c.width, c.height], float)


def gen_rng(out: dict) -> None:
    parts = [(0,), (7,), (0, "init-params"), (0, 3, "light-select"),
             (5, 2, 1, "targets"), ("primary",), (123456789012345, -3, "x"),
             (2**64 - 1, 2**63)]
    keys = np.array([R.stream_key(*p) for p in parts], dtype=np.uint64)
    out["rng_keys"] = keys
    out["rng_parts"] = np.array([repr(p) for p in parts])
    # first 41 doubles (crosses a Philox block boundary at an odd offset)
    out["rng_first"] = np.stack([R.stream(*p).random(41) for p in parts])
    raw = R.stream(0, 3, "light-select").bit_generator.random_raw(16)
    out["rng_raw"] = np.asarray(raw, dtype=np.uint64)
    # uniform(lo, hi) over a broadcast (n,3) shape, row-major
    g = R.stream(9, 1, 0, "world-samples")
    out["rng_uniform"] = g.uniform(np.array([-3.0, 0.0, -2.2]), np.array([3.0, 1.5, 3.0]),
                                   size=(5, 3))
    # random access: draws 1001..1010 of a stream
    g = R.stream(0, 3, "light-select")
    g.random(1001)
    out["rng_at1001"] = g.random(10)


def gen_scenes(out: dict) -> None:
    for name, d in (("boxes8", boxes_scene(8)), ("boxes32", boxes_scene(32)),
                    ("rooms128", rooms_scene(128)), ("pbox8", point_light_dict(8))):
        scene_arrays(name + "_", scene_from_dict(d), out)


def gen_hashgrid(out: dict, tag: str, levels: int, tsize: int, seed: int) -> None:
    s = scene_from_dict(boxes_scene(32))
    cfg = HashGridConfig(levels=levels, table_size=tsize, features_per_level=2,
                         aabb_min=s.aabb_min, aabb_max=s.aabb_max)
    g = R.stream(seed, "golden-pos")
    n = 1500
    pos = g.uniform(s.aabb_min - 0.3, s.aabb_max + 0.3, size=(n, 3))
    pos[:8] = [[-3, 0, -2.2], [3, 1.5, 3], [0, 0, 0], [3.0, 0.0, -2.2],
               [-3.5, 2.0, 4.0], [0.123456789, 1.2, 0.5], [1e-17, 1.5, 3.0], [2.9999999999, 0.75, 0.4]]
    table = VisibilityCache(MODE_LIGHTS, 4, cfg, seed=seed).grid_params
    feats, ctx = encode_batch(pos, cfg, table)
    q = _normalize(cfg, pos)
    idx = np.stack([_level_lookup(cfg, l, q)[0] for l in range(levels)], axis=1)
    w = np.stack([_level_lookup(cfg, l, q)[1] for l in range(levels)], axis=1)
    up = g.standard_normal((n, cfg.output_dim)).astype(np.float32)
    grad = grad_from_ctx(cfg, ctx, up, dtype=np.float32)
    nz = np.flatnonzero(grad.reshape(-1))
    out[tag + "_pos"] = pos
    out[tag + "_res"] = np.array([cfg.resolution(l) for l in range(levels)])
    out[tag + "_dense"] = np.array([cfg.dense(l) for l in range(levels)])
    out[tag + "_idx"] = idx.astype(np.int32)
    out[tag + "_w"] = w
    out[tag + "_feats"] = feats
    out[tag + "_table_sha"] = np.array(sha(table))
    out[tag + "_up"] = up
    out[tag + "_grad_nz"] = nz.astype(np.int64)
    out[tag + "_grad_val"] = grad.reshape(-1)[nz]


def gen_mlp(out: dict) -> None:
    cfg = MLPConfig(input_dim=16, output_dim=8, hidden_dims=(64, 64))
    g = R.stream(3, "golden-mlp")
    params = he_init(cfg, g)
    x = (g.standard_normal((256, 16)) * 1e-2).astype(np.float32)
    t = (g.random((256, 8)) < 0.5).astype(np.float32)
    y, cache = forward(params, cfg, x)
    loss = l2_loss(y, t)
    grads, d_in = backward_l2(params, cfg, cache, t)
    for i, (wt, bs) in enumerate(zip(params.weights, params.biases)):
        out[f"mlp_w{i}"] = wt
        out[f"mlp_b{i}"] = bs
        out[f"mlp_gw{i}"] = grads.weights[i]
        out[f"mlp_gb{i}"] = grads.biases[i]
    out["mlp_x"] = x
    out["mlp_t"] = t
    out["mlp_y"] = y
    out["mlp_loss"] = np.array(loss)
    out["mlp_dx"] = d_in
    # 3 Adam steps over a flat float32 vector with given grads and lrs
    p0 = g.standard_normal(1000).astype(np.float32)
    gs = [(g.standard_normal(1000) * 10.0 ** g.integers(-8, 0, 1000)).astype(np.float32)
          for _ in range(3)]
    gs[1][::7] = 0.0
    lrs = [0.05, 0.04975, 0.0495]
    p = {"p": p0.copy()}
    st = AdamState.for_params(p)
    traj = []
    for gi, lr in zip(gs, lrs):
        adam_step(p, {"p": gi}, st, lr)
        traj.append(p["p"].copy())
    out["adam_p0"] = p0
    out["adam_g"] = np.stack(gs)
    out["adam_lr"] = np.array(lrs)
    out["adam_traj"] = np.stack(traj)
    out["adam_m"] = st.m["p"]
    out["adam_v"] = st.v["p"]


def gen_sampling(out: dict) -> None:
    g = R.stream(11, "golden-wrs")
    w = g.random((512, 32)) * (g.random((512, 32)) < 0.4)
    w[0] = 0.0
    w[1] = 0.0
    w[1, 31] = 2.5
    w[2, :] = 1.0
    rs = R.stream(0, 4, "light-select")
    idx, w_sel, w_sum = wrs_select_batch(w, rs)
    idx2, _, _ = wrs_select_batch(w[:17], rs)   # stream continues
    out["wrs_w"] = w
    out["wrs_idx"] = idx
    out["wrs_wsel"] = w_sel
    out["wrs_wsum"] = w_sum
    out["wrs_idx2"] = idx2

    s = scene_from_dict(boxes_scene(32))
    cam = Camera(position=s.camera.position, look_at=s.camera.look_at, up=s.camera.up,
                 fov_deg=s.camera.fov_deg, width=40, height=24)
    gb = make_gbuffer(s, cam)
    ctx = PixelCtx(s, gb.flat("position"), gb.flat("normal"), gb.flat("albedo"))
    for k in ("hit", "position", "normal", "albedo", "depth", "light_id", "emissive"):
        out["gb_" + k] = gb.flat(k)
    out["nls_factor"] = ctx.factor_matrix()
    out["nls_lum"] = ctx.lum_matrix()
    vis = g.random((ctx.n, 32)).astype(np.float32)
    vis[::5] = 0.5

    class Fixed:
        mode = MODE_LIGHTS
        output_dim = 32

        def infer(self, positions):
            return vis[: positions.shape[0]]

    ids, pts, big_w = nls_sample_batch(ctx, Fixed(), R.stream(0, 7, "light-select"))
    out["nls_vis"] = vis
    out["nls_ids"] = ids
    out["nls_pts"] = pts
    out["nls_W"] = big_w
    ids_b, pts_b, w_b = nls_sample_batch(ctx, Fixed(), R.stream(0, 7, "light-select"), 0.0)
    out["nls_ids_biased"] = ids_b
    out["nls_W_biased"] = w_b
    out["ndi_rgb"] = neural_di_batch(ctx, Fixed())

    # full 64x64 G-buffer of the C1 point-light scene (exercises POINT factors)
    sp = scene_from_dict(point_light_dict(8))
    gbp = make_gbuffer(sp)
    ctxp = PixelCtx(sp, gbp.flat("position"), gbp.flat("normal"), gbp.flat("albedo"))
    out["pgb_position"] = gbp.flat("position")
    out["pgb_normal"] = gbp.flat("normal")
    out["pgb_albedo"] = gbp.flat("albedo")
    out["pgb_hit"] = gbp.flat("hit")
    out["pgb_factor"] = ctxp.factor_matrix()


def gen_shade(out: dict) -> None:
    """render.py:220-246 (shade_batch) on a boxes32 G-buffer with random
    (id, point, W) samples -- ids include -1, W includes 0 -- on the C1
    point-light G-buffer, and on the NLS samples of gen_sampling's fixture."""
    g = R.stream(3, "golden-shade")
    s = scene_from_dict(boxes_scene(32))
    cam = Camera(position=s.camera.position, look_at=s.camera.look_at, up=s.camera.up,
                 fov_deg=s.camera.fov_deg, width=64, height=40)
    gb = make_gbuffer(s, cam)
    pos, nrm, alb = gb.flat("position"), gb.flat("normal"), gb.flat("albedo")
    n = pos.shape[0]
    ids = g.integers(-1, s.n_lights, size=n)
    pts = s.light_points(np.maximum(ids, 0), g.random((n, 2)))
    big_w = g.random(n) * 40.0 * (g.random(n) < 0.9)
    out["b32_position"], out["b32_normal"], out["b32_albedo"] = pos, nrm, alb
    out["b32_ids"], out["b32_pts"], out["b32_W"] = ids, pts, big_w
    out["b32_rgb"] = shade_batch(s, pos, nrm, alb, ids, pts, big_w)

    sp = scene_from_dict(point_light_dict(8))
    gbp = make_gbuffer(sp)
    pos, nrm, alb = gbp.flat("position"), gbp.flat("normal"), gbp.flat("albedo")
    n = pos.shape[0]
    ids = g.integers(-1, sp.n_lights, size=n)
    pts = sp.light_points(np.maximum(ids, 0), g.random((n, 2)))
    big_w = g.random(n) * 8.0
    out["p8_ids"], out["p8_pts"], out["p8_W"] = ids, pts, big_w
    out["p8_rgb"] = shade_batch(sp, pos, nrm, alb, ids, pts, big_w)

    smp = np.load(os.path.join(HERE, "sampling.npz"))
    out["nls_rgb"] = shade_batch(s, smp["gb_position"], smp["gb_normal"], smp["gb_albedo"], smp["nls_ids"],
                                 smp["nls_pts"], smp["nls_W"])


def gen_snapshot(out: dict) -> None:
    """A VCSNAP1 file written by the reference cache after two train steps (cache.py:77-117),
    plus its infer() output on fixed positions -- pins on-disk interop both ways."""
    s = scene_from_dict(boxes_scene(8))
    cfg = HashGridConfig(levels=4, table_size=1 << 10, features_per_level=2, aabb_min=s.aabb_min,
                         aabb_max=s.aabb_max)
    c = VisibilityCache(MODE_LIGHTS, 8, cfg, seed=4)
    g = R.stream(9, "golden-snapshot")
    pos = g.uniform(s.aabb_min, s.aabb_max, (64, 3))
    for _ in range(2):
        c.train_step(pos, (g.random((64, 8)) < 0.5).astype(np.float32))
    path = os.path.join(HERE, "ref_snapshot.vcsnap")
    c.save(path)
    q = g.uniform(s.aabb_min, s.aabb_max, (257, 3))
    out["snap_pos"] = q
    out["snap_infer"] = c.infer(q)
    out["snap_step"] = np.array(c.step)


def gen_clusters(out: dict) -> None:
    """Clustered NVC (sampling.py:252-359, training.py:121-128): k-means on the
    rooms scenes' lights, cluster shadow-ray targets, and the two-step sampler
    with a fixed cluster-visibility cache."""
    from viscache.sampling import clustered_sample_batch, kmeans_cluster
    for tag, n_lights, k in (("r128k16", 128, 16), ("r1024k32", 1024, 32), ("b32k8", 32, 8), ("b8k8", 8, 8)):
        s = scene_from_dict(rooms_scene(n_lights) if tag.startswith("r") else boxes_scene(n_lights))
        cs = kmeans_cluster(s.lights, k, R.stream(0, R.CLUSTERING))
        out[f"km_{tag}_centroids"] = cs.centroids
        out[f"km_{tag}_sizes"] = np.array([mem.size for mem in cs.members])
        out[f"km_{tag}_members"] = np.concatenate(cs.members)
        out[f"km_{tag}_history"] = np.array(cs.inertia_history)
    # targets: rooms128 with 16 clusters, a few hundred rows
    s = scene_from_dict(rooms_scene(128))
    cs = kmeans_cluster(s.lights, 16, R.stream(0, R.CLUSTERING))
    g = R.stream(5, "golden-cluster-pos")
    pos = g.uniform(s.aabb_min, s.aabb_max, (777, 3))
    out["ct_pos"] = pos
    out["ct_tgt"] = compute_visibility_targets(pos, s, R.stream(0, 2, 0, R.TARGETS), clusters=cs)
    # two-step sampler on a 48x32 rooms128 G-buffer with fixed cluster visibilities
    cam = Camera(position=s.camera.position, look_at=s.camera.look_at, up=s.camera.up,
                 fov_deg=s.camera.fov_deg, width=48, height=32)
    gb = make_gbuffer(s, cam)
    ctx = PixelCtx(s, gb.flat("position"), gb.flat("normal"), gb.flat("albedo"))
    vis = g.random((ctx.n, 16)).astype(np.float32)
    vis[::7] = 0.25

    class Fixed:
        mode = "clusters"
        output_dim = 16

        def infer(self, positions):
            return vis[: positions.shape[0]]

    ids, pts, big_w = clustered_sample_batch(ctx, Fixed(), cs, R.stream(0, 3, R.LIGHT_SELECT))
    out["cs_vis"] = vis
    out["cs_ids"], out["cs_pts"], out["cs_W"] = ids, pts, big_w
    for k in ("position", "normal", "albedo"):
        out["cs_gb_" + k] = gb.flat(k)


def gen_training(out: dict) -> None:
    s8 = scene_from_dict(boxes_scene(8))
    pts = gen_screen_samples(s8, s8.camera, 256, R.stream(6))
    out["screen_boxes8_256"] = pts

    sp = scene_from_dict(point_light_dict(8))
    key = (0, 0, 0)
    world = gen_world_samples(sp, 4096, R.stream(*key, R.WORLD_SAMPLES))
    screen = gen_screen_samples(sp, sp.camera, 4096, R.stream(*key, R.SCREEN_SAMPLES))
    pos = np.concatenate([world, screen])
    tgt = compute_visibility_targets(pos, sp, R.stream(*key, R.TARGETS))
    out["c1_pos"] = pos
    out["c1_tgt"] = tgt.astype(np.uint8)

    s32 = scene_from_dict(boxes_scene(32))
    key = (0, 3, 0)
    world = gen_world_samples(s32, 2048, R.stream(*key, R.WORLD_SAMPLES))
    screen = gen_screen_samples(s32, s32.camera, 2048, R.stream(*key, R.SCREEN_SAMPLES))
    pos = np.concatenate([world, screen])
    tgt = compute_visibility_targets(pos, s32, R.stream(*key, R.TARGETS))
    out["b32_pos"] = pos
    out["b32_tgt"] = tgt.astype(np.uint8)

    # penumbra visibility for hand-picked segments (degenerate + grazing)
    x = np.array([[0.0, 0.0, 0.0], [2.0, 0.0, 2.0], [0.0, 1.35 - 1e-6, 0.0], [-3.0, 0.0, -2.2]])
    y = np.array([[0.0, 1.35, 0.0], [-2.1, 1.35, -1.3], [0.0, 1.35, 0.0], [3.0, 1.5, 3.0]])
    out["vis_x"] = x
    out["vis_y"] = y
    out["vis_b32"] = visibility_batch(s32.bvh, x, y)


def c1_cache(scene, dtype=np.float32, seed=0):
    cfg = HashGridConfig(levels=8, table_size=1 << 14, features_per_level=2,
                         aabb_min=scene.aabb_min, aabb_max=scene.aabb_max)
    return widened_cache(scene.n_lights, cfg, (64, 64), seed, dtype)


def widened_cache(k, cfg, hidden, seed=0, dtype=np.float32):
    """Reference cache with a non-default MLP width.  The reference hardcodes
    (32,32) (cache.py:37-38); the generalisation keeps its single init stream:
    table first, then He weights of the configured topology (cache.py:41-43)."""
    c = VisibilityCache(MODE_LIGHTS, k, cfg, seed=seed, dtype=dtype)
    g = R.stream(seed, R.INIT_PARAMS)
    c.grid_params = init_params(cfg, g, dtype=dtype)
    c.net_cfg = MLPConfig(input_dim=cfg.output_dim, output_dim=k, hidden_dims=hidden)
    c.net_params = he_init(c.net_cfg, g, dtype=dtype)
    c.adam = AdamState.for_params(c._param_dict())
    return c


def gen_curves(out: dict, quick: bool) -> None:
    sp = scene_from_dict(point_light_dict(8))
    cfg = TrainFrameConfig()
    frames = 6 if quick else 20
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        c = c1_cache(sp, dt)
        losses = [train_frame(sp, sp.camera, c, cfg, frame=f) for f in range(frames)]
        out["c1_loss_" + tag] = np.array(losses)
        if dt is np.float32:
            out["c1_final_grid_sha"] = np.array(sha(c.grid_params))
            # visibility of the trained cache on fixed probes (mean-abs compare)
            probes = R.stream(0, "probes").uniform(sp.aabb_min, sp.aabb_max, (256, 3))
            out["c1_probe_pos"] = probes
            out["c1_probe_vis"] = c.infer(probes)
    # first-step exact state (one train_step on the frame-0 batch)
    c = c1_cache(sp)
    loss0 = c.train_step(out["c1_pos"], out["c1_tgt"].astype(np.float32))
    out["c1_step0_loss"] = np.array(loss0)
    out["c1_step0_w0"] = c.net_params.weights[0]
    out["c1_step0_b2"] = c.net_params.biases[2]
    # determinism config from the reference suite (levels=4, T=2^10, 64+64, seed 5)
    pen = {
        "camera": {"position": [0, 1.6, 3.2], "look_at": [0, 0, 0], "up": [0, 1, 0],
                   "fov_deg": 55.0, "width": 96, "height": 54},
        "materials": [{"albedo": [0.7, 0.7, 0.7]}, {"albedo": [0.5, 0.3, 0.3]}],
        "meshes": [{"material": 0, "triangles": [[[-4, 0, -4], [4, 0, -4], [4, 0, 4]],
                                                 [[-4, 0, -4], [4, 0, 4], [-4, 0, 4]]]},
                   {"material": 1, "triangles": [[[-.5, 1, -.5], [.5, 1, -.5], [.5, 1, .5]],
                                                 [[-.5, 1, -.5], [.5, 1, .5], [-.5, 1, .5]]]}],
        "lights": [{"type": "rect", "corner": [-0.4, 2.0, -0.4], "edge_u": [0.8, 0, 0],
                    "edge_v": [0, 0, 0.8], "radiance": [10.0, 10.0, 10.0]}],
    }
    ps = scene_from_dict(pen)
    c = VisibilityCache(MODE_LIGHTS, 1, HashGridConfig(levels=4, table_size=1 << 10,
                                                       aabb_min=ps.aabb_min,
                                                       aabb_max=ps.aabb_max), seed=5)
    tcfg = TrainFrameConfig(n_world=64, n_screen=64, seed=5)
    out["pen_loss"] = np.array([train_frame(ps, ps.camera, c, tcfg, frame=f) for f in range(3)])
    # C2 settings (boxes32, L=16 T=2^19 F=2, 3x64) — a few frames at full batch
    if not quick:
        s32 = scene_from_dict(boxes_scene(32))
        cfg2 = HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2,
                              aabb_min=s32.aabb_min, aabb_max=s32.aabb_max)
        c2 = widened_cache(32, cfg2, (64, 64, 64))
        out["c2_loss_f32"] = np.array([train_frame(s32, s32.camera, c2, cfg, frame=f)
                                       for f in range(6)])


def gen_long_curves(out: dict) -> None:
    """Headline-config loss curves (north_star: "the loss curve over N online
    frames stays within tolerance"): C2 = boxes32, L=16 T=2^19 F=2, MLP 3x64,
    K=32, 60 online frames (BASELINE configs[1]), run by the reference at
    float32 and float64 (the f32-vs-f64 spread calibrates the tolerance); C4 =
    rooms128, 3x128 MLP, K=128, 8 frames at both dtypes.  Also the trained C2
    cache's visibility on fixed probes (mean-abs compare only: SURVEY 8(c))."""
    cfg = TrainFrameConfig()
    s32 = scene_from_dict(boxes_scene(32))
    g2 = HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2,
                        aabb_min=s32.aabb_min, aabb_max=s32.aabb_max)
    probes = R.stream(0, "probes").uniform(s32.aabb_min, s32.aabb_max, (4096, 3))
    out["c2_probe_pos"] = probes
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        c2 = widened_cache(32, g2, (64, 64, 64), dtype=dt)
        out["c2_loss60_" + tag] = np.array([train_frame(s32, s32.camera, c2, cfg, frame=f) for f in range(60)])
        out["c2_probe_vis_" + tag] = c2.infer(probes)
        print("c2", tag, out["c2_loss60_" + tag][[0, 1, 10, 59]], flush=True)
    # reference-trained C1 cache (20 frames, f32): its parameters and its own
    # visibility on fixed probes, so the GPU inference paths can be checked
    # against the reference at trained scale (not only at init)
    sp = scene_from_dict(point_light_dict(8))
    c1 = c1_cache(sp)
    for f in range(20):
        train_frame(sp, sp.camera, c1, cfg, frame=f)
    out["c1t_grid"] = c1.grid_params
    for i, (w, b) in enumerate(zip(c1.net_params.weights, c1.net_params.biases)):
        out[f"c1t_w{i}"] = w
        out[f"c1t_b{i}"] = b
    p1 = R.stream(0, "probes").uniform(sp.aabb_min, sp.aabb_max, (4096, 3))
    gb = make_gbuffer(sp, sp.camera)
    p1 = np.concatenate([p1, gb.flat("position")[gb.flat("hit")]])
    out["c1t_probe_pos"] = p1
    out["c1t_probe_vis"] = c1.infer(p1)
    r128 = scene_from_dict(rooms_scene(128))
    g4 = HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2,
                        aabb_min=r128.aabb_min, aabb_max=r128.aabb_max)
    for dt, tag in ((np.float32, "f32"), (np.float64, "f64")):
        c4 = widened_cache(128, g4, (128, 128, 128), dtype=dt)
        out["c4_loss_" + tag] = np.array([train_frame(r128, r128.camera, c4, cfg, frame=f) for f in range(8)])
        print("c4", tag, out["c4_loss_" + tag], flush=True)


class WaveCache:
    """Deterministic stand-in cache (the reference's FixedCache pattern,
    test_sampling.py:21-30): visibility = 0.5 + 0.4 sin(a . pos + j)."""
    mode = MODE_LIGHTS

    def __init__(self, k):
        self.output_dim = k

    def infer(self, positions):
        pos = np.atleast_2d(np.asarray(positions, np.float64))
        ph = pos @ np.array([1.3, 2.1, 0.7])
        return (0.5 + 0.4 * np.sin(ph[:, None] + np.arange(self.output_dim))).astype(np.float32)


def gen_scalar(out: dict) -> None:
    """Scalar API wrappers (sampling.py:88-101,141-176,208-222): wrs_select,
    nls_sample, neural_di_shade, unshadowed_weight, unshadowed_rgb_one and
    PixelCtx.phat_ids on 48 shading points of boxes8 (rect lights) and 16 of
    the point-light C1 scene."""
    from viscache.sampling import (ShadingPoint, neural_di_shade, nls_sample, unshadowed_rgb_one,
                                   unshadowed_weight, wrs_select)
    g = np.random.default_rng(21)
    rows = []
    for tag, sc, n in (("b8", scene_from_dict(boxes_scene(8)), 48), ("p8", scene_from_dict(point_light_dict(8)), 16)):
        cam = Camera(position=sc.camera.position, look_at=sc.camera.look_at, up=sc.camera.up,
                     fov_deg=sc.camera.fov_deg, width=40, height=24)
        gb = make_gbuffer(sc, cam)
        hit = np.flatnonzero(gb.flat("hit"))
        pick = hit[g.choice(hit.size, n, replace=False)]
        pos, nrm, alb = (gb.flat(k)[pick] for k in ("position", "normal", "albedo"))
        out[f"sc_{tag}_pos"], out[f"sc_{tag}_nrm"], out[f"sc_{tag}_alb"] = pos, nrm, alb
        k = sc.n_lights
        cache = WaveCache(k)
        wts = g.random((n, 6)) * (g.random((n, 6)) < 0.7)
        out[f"sc_{tag}_wrs_w"] = wts
        res, nls, ndi, uw, urgb = [], [], [], [], []
        for i in range(n):
            sp = ShadingPoint(position=pos[i], normal=nrm[i], albedo=alb[i])
            r = wrs_select(wts[i], R.stream(0, i, "wrs-scalar"))
            res.append([r.y, r.w_y, r.w_sum, r.M, r.W])
            lid, pt, big_w = nls_sample(sp, cache, sc, R.stream(1, i, "light-select"))
            nls.append([lid, *pt, big_w])
            ndi.append(neural_di_shade(sp, cache, sc))
            uw.append([unshadowed_weight(sp, j, sc) for j in range(k)])
            urgb.append([unshadowed_rgb_one(sp, j, sc) for j in range(k)])
        out[f"sc_{tag}_wrs"] = np.array(res, float)
        out[f"sc_{tag}_nls"] = np.array(nls, float)
        out[f"sc_{tag}_ndi"] = np.array(ndi)
        out[f"sc_{tag}_uw"] = np.array(uw)
        out[f"sc_{tag}_urgb"] = np.array(urgb)
        ctx = PixelCtx(sc, pos, nrm, alb)
        ids = g.integers(-1, k, n)
        out[f"sc_{tag}_phat_ids"] = ids
        out[f"sc_{tag}_phat"] = ctx.phat_ids(ids)


def gen_restir(out: dict) -> None:
    """RIS / ReSTIR baselines (sampling.py:369-637) on boxes8 at 48x32: two RIS
    frames (the first on a stream whose integers() left a kept 32-bit half),
    temporal merges in both clamp modes (one with a partly invalid history),
    spatial reuse at radius 32 and 4, clustered initial reservoirs; plus the
    next draws of each stream (the continuation)."""
    from viscache.sampling import (ReservoirGrid, cnvc_initial_batch, kmeans_cluster, restir_spatial_batch,
                                   restir_temporal_batch, ris_initial_batch)
    s = scene_from_dict(boxes_scene(8))
    cam = Camera(position=s.camera.position, look_at=s.camera.look_at, up=s.camera.up,
                 fov_deg=s.camera.fov_deg, width=48, height=32)
    gb = make_gbuffer(s, cam)
    ctx = PixelCtx(s, gb.flat("position"), gb.flat("normal"), gb.flat("albedo"))

    def save(tag, g, rng=None):
        for k in ("y", "point", "w_y", "w_sum", "M", "W", "valid"):
            out[f"{tag}_{k}"] = np.asarray(getattr(g, k))
        if rng is not None:
            out[f"{tag}_next"] = rng.random(3)

    r0 = R.stream(0, 0, "restir-initial")
    out["pre_ints"] = r0.integers(0, 7, size=3)
    g0 = ris_initial_batch(ctx, r0, 8)
    save("ris0", g0, r0)
    r1 = R.stream(0, 1, "restir-initial")
    g1 = ris_initial_batch(ctx, r1, 8)
    save("ris1", g1, r1)
    rt = R.stream(0, 1, "restir-temporal")
    t_m = restir_temporal_batch(g1, g0, ctx, rt, 20.0, "m")
    save("tm", t_m, rt)
    g0b = ReservoirGrid(g0.n)
    for k in ("y", "point", "w_y", "w_sum", "M", "W", "valid"):
        setattr(g0b, k, np.array(getattr(g0, k)))
    g0b.valid[::3] = False
    g0b.M[1::5] = 60.0
    rt2 = R.stream(0, 2, "restir-temporal")
    t_c = restir_temporal_batch(g1, g0b, ctx, rt2, 2.0, "contribution")
    save("tc", t_c, rt2)
    rt3 = R.stream(0, 3, "restir-temporal")
    save("tm2", restir_temporal_batch(g1, g0b, ctx, rt3, 2.0, "m"), rt3)
    for rad in (32, 4):
        rs = R.stream(0, rad, "restir-spatial")
        sp = restir_spatial_batch(t_m, ctx, gb.shape, gb.flat("hit"), gb.flat("depth"), ctx.normals, rs, rad, 4)
        save(f"sp{rad}", sp, rs)
    cl = kmeans_cluster(s.lights, 4, R.stream(0, "clustering"))
    rc = R.stream(0, 2, "restir-initial")
    save("cn", cnvc_initial_batch(ctx, WaveCache(4), cl, rc), rc)


def main() -> None:
    quick = "--quick" in sys.argv
    groups = {
        "rng": gen_rng, "scenes": gen_scenes, "mlp": gen_mlp,
        "sampling": gen_sampling, "training": gen_training, "shade": gen_shade, "snapshot": gen_snapshot,
        "clusters": gen_clusters, "curves": gen_long_curves, "scalar": gen_scalar, "restir": gen_restir,
    }
    only = [a for a in sys.argv[1:] if not a.startswith("-")]
    if only:   # regenerate just the named groups, e.g. `make_golden.py shade`
        for name in only:
            out = {}
            groups[name](out)
            np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
            print("wrote", name)
        return
    for name, fn in groups.items():
        out: dict = {}
        fn(out)
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print("wrote", name, sorted(out)[:6], "...")
    out = {}
    gen_hashgrid(out, "hc1", 8, 1 << 14, 0)
    gen_hashgrid(out, "hc2", 16, 1 << 19, 1)
    np.savez_compressed(os.path.join(HERE, "hashgrid.npz"), **out)
    print("wrote hashgrid")
    tr = dict(np.load(os.path.join(HERE, "training.npz")))
    gen_curves(tr, quick)
    np.savez_compressed(os.path.join(HERE, "training.npz"), **tr)
    print("wrote curves")


if __name__ == "__main__":
    main()
