"""GPU parity: every CUDA entry point against the oracle and the reference's
golden vectors.  Bit-exact where the reference is integer/index work or
FP64 with a pinned op order; explicit tolerances otherwise (stated inline)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import vc_oracle as O  # noqa: E402
from paper_2506_05930_b200 import (PRECISION_FP16, PRECISION_FP32, HashGridConfig,  # noqa: E402
                                   MODE_LIGHTS, PixelCtx, VisibilityCache, make_gbuffer,
                                   nls_sample_batch, neural_di_batch, scene_from_dict, train_frame,
                                   TrainFrameConfig, wrs_select_batch)
from paper_2506_05930_b200 import rng as R  # noqa: E402
from paper_2506_05930_b200 import _lib  # noqa: E402
from paper_2506_05930_b200.scenes import boxes_point_scene, boxes_scene, rooms_scene  # noqa: E402
from paper_2506_05930_b200.training import (compute_visibility_targets, gen_screen_samples,  # noqa: E402
                                            gen_world_samples)

DEV = torch.device("cuda", 0)
FP16_VIS_TOL = 4e-3     # fp16 table + fp16 weights/activations, fp32 accumulate


@pytest.fixture(scope="module")
def boxes32():
    return scene_from_dict(boxes_scene(32))


@pytest.fixture(scope="module")
def boxes8():
    return scene_from_dict(boxes_scene(8))


@pytest.fixture(scope="module")
def pbox8():
    return scene_from_dict(boxes_point_scene(8))


def grid_cfg(scene, levels, tsize):
    return HashGridConfig(levels=levels, table_size=tsize, features_per_level=2,
                          aabb_min=scene.aabb_min, aabb_max=scene.aabb_max)


# ---------------------------------------------------------------------------
# RNG + WRS
# ---------------------------------------------------------------------------
class TestWrs:
    def test_wrs_bit_exact_vs_reference(self, g_samp):
        rs = R.stream(0, 4, "light-select")
        idx, wsel, wsum = wrs_select_batch(g_samp["wrs_w"], rs)
        np.testing.assert_array_equal(idx, g_samp["wrs_idx"])
        np.testing.assert_array_equal(wsel, g_samp["wrs_wsel"])
        np.testing.assert_array_equal(wsum, g_samp["wrs_wsum"])
        idx2, _, _ = wrs_select_batch(g_samp["wrs_w"][:17], rs)       # stream continues
        np.testing.assert_array_equal(idx2, g_samp["wrs_idx2"])

    @pytest.mark.parametrize("k,offset", [(1, 0), (3, 5), (32, 1), (128, 7), (7, 2**33 + 3)])
    def test_wrs_matches_oracle_any_offset(self, k, offset):
        g = np.random.default_rng(k)
        w = g.random((999, k)) * (g.random((999, k)) < 0.5)
        key = R.stream_key(9, k, "light-select")
        idx, wsel, wsum = wrs_select_batch(w, R.Stream(key=key, offset=offset))
        oi, ow, os_ = O.wrs_select(w, key, offset)
        np.testing.assert_array_equal(idx, oi)
        np.testing.assert_array_equal(wsel, ow)
        np.testing.assert_array_equal(wsum, os_)


# ---------------------------------------------------------------------------
# encoder
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("tag,levels,tsize,seed", [("hc1", 8, 1 << 14, 0), ("hc2", 16, 1 << 19, 1)])
def test_encoder_bit_exact(g_hash, boxes32, tag, levels, tsize, seed):
    c = VisibilityCache(MODE_LIGHTS, 4, grid_cfg(boxes32, levels, tsize), seed=seed)
    feats, idx, w = c.encode(g_hash[tag + "_pos"], with_ctx=True)
    np.testing.assert_array_equal(idx, g_hash[tag + "_idx"])
    np.testing.assert_array_equal(w, g_hash[tag + "_w"])
    np.testing.assert_array_equal(feats, g_hash[tag + "_feats"])


# ---------------------------------------------------------------------------
# inference: fp32 SIMT parity path and the tcgen05 fused path
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("levels,tsize,hidden,k,f", [(8, 1 << 14, (64, 64), 8, 2), (16, 1 << 19, (64, 64, 64), 32, 2),
                                                     (4, 1 << 10, (32, 32), 1, 2),
                                                     (16, 1 << 19, (128, 128, 128), 128, 2),
                                                     (10, 1 << 14, (32, 32), 5, 4), (3, 1 << 8, (24, 40), 3, 1)])
def test_infer_vs_oracle(boxes32, levels, tsize, hidden, k, f):
    cfg = HashGridConfig(levels=levels, table_size=tsize, features_per_level=f,
                         aabb_min=boxes32.aabb_min, aabb_max=boxes32.aabb_max)
    c = VisibilityCache(MODE_LIGHTS, k, cfg, seed=3, hidden_dims=hidden)
    oc = O.Cache(O.Grid(levels=levels, features_per_level=f, table_size=tsize, aabb_min=boxes32.aabb_min,
                        aabb_max=boxes32.aabb_max), k, hidden=hidden, seed=3)
    np.testing.assert_array_equal(c.grid_params, oc.table)
    pos = np.random.default_rng(1).uniform(boxes32.aabb_min - 0.1, boxes32.aabb_max + 0.1, (3001, 3))
    want = oc.infer(pos)
    got32 = c.infer(pos, precision=PRECISION_FP32)
    np.testing.assert_allclose(got32, want, rtol=0, atol=1e-6)
    got16 = c.infer(pos, precision=PRECISION_FP16)
    assert np.abs(got16 - want).max() < FP16_VIS_TOL


@pytest.mark.parametrize("variant", ["ts", "NVC_MLP_QUADS"])
def test_c4_mlp_takes_the_tcgen05_path(boxes32, variant, monkeypatch):
    """C4's 3x128 MLP with 128 outputs runs on the tcgen05 kernels -- TS mode (two
    warpgroups x 192 TMEM columns) and SS mode (two tiles in flight so the
    activation tiles fit in smem) -- not the fp32 fallback."""
    if variant != "ts":
        monkeypatch.setenv(variant, "1")
    cfg = grid_cfg(boxes32, 16, 1 << 19)
    c = VisibilityCache(MODE_LIGHTS, 128, cfg, seed=3, hidden_dims=(128, 128, 128))
    oc = O.Cache(O.Grid(levels=16, features_per_level=2, table_size=1 << 19, aabb_min=boxes32.aabb_min,
                        aabb_max=boxes32.aabb_max), 128, hidden=(128, 128, 128), seed=3)
    pos = np.random.default_rng(4).uniform(boxes32.aabb_min, boxes32.aabb_max, (70001, 3))
    pt = torch.from_numpy(pos).to(DEV)
    out = torch.empty((pos.shape[0], 128), dtype=torch.float32, device=DEV)
    _lib.call("nvc_infer", c.model, pt.data_ptr(), pos.shape[0], PRECISION_FP16, out.data_ptr(),
              _lib.ptr(c.query_workspace(pos.shape[0])), _lib.stream_ptr())      # raises if unsupported
    assert np.abs(out.cpu().numpy() - oc.infer(pos)).max() < FP16_VIS_TOL


@pytest.mark.parametrize("levels,tsize,hidden", [(8, 1 << 14, (32, 32)), (16, 1 << 19, (64, 64, 64))])
def test_f4_encoder_equals_generic(boxes32, levels, tsize, hidden, monkeypatch):
    """F = 4 grids (the reference's default features_per_level; the clustered
    preset is L=8, T=2^14): the 16-byte-gather encoder k_enc_tiles4 gives the
    same fp16 query outputs, bit for bit, as the generic per-half encoder, on
    N(0, 0.3) tables; and both stay within the fp16 tolerance of the oracle."""
    cfg = HashGridConfig(levels=levels, table_size=tsize, features_per_level=4, aabb_min=boxes32.aabb_min,
                         aabb_max=boxes32.aabb_max)
    c = VisibilityCache(MODE_LIGHTS, 32, cfg, seed=2, hidden_dims=hidden)
    c.grid_params = (np.random.default_rng(6).standard_normal(c.grid_params.shape) * 0.3).astype(np.float32)
    pos = np.random.default_rng(7).uniform(boxes32.aabb_min, boxes32.aabb_max, (50003, 3))
    fast = c.infer(pos, precision=PRECISION_FP16)
    monkeypatch.setenv("NVC_ENC_GENERIC", "1")
    generic = c.infer(pos, precision=PRECISION_FP16)
    np.testing.assert_array_equal(fast, generic)
    ref = c.infer(pos, precision=PRECISION_FP32)
    assert np.abs(fast.astype(np.float64) - ref).max() < 2e-2


def test_infer_trained_weights_fp16(boxes32):
    """fp16 tolerance also holds away from init (trained-scale weights)."""
    cfg = grid_cfg(boxes32, 16, 1 << 19)
    c = VisibilityCache(MODE_LIGHTS, 32, cfg, seed=0, hidden_dims=(64, 64, 64))
    g = np.random.default_rng(2)
    table = (g.standard_normal(c.grid_params.shape) * 0.3).astype(np.float32)
    c.grid_params = table
    pos = g.uniform(boxes32.aabb_min, boxes32.aabb_max, (2048, 3))
    a, b = c.infer(pos, precision=PRECISION_FP32), c.infer(pos, precision=PRECISION_FP16)
    assert np.abs(a - b).max() < 2e-2 and np.abs(a - b).mean() < 2e-3


def test_infer_rejects_nonfinite(boxes32):
    c = VisibilityCache(MODE_LIGHTS, 4, grid_cfg(boxes32, 4, 1 << 10))
    with pytest.raises(ValueError):
        c.infer(np.array([[0.0, np.nan, 0.0]]))


def test_infer_empty_and_ragged(boxes32):
    c = VisibilityCache(MODE_LIGHTS, 8, grid_cfg(boxes32, 8, 1 << 14), hidden_dims=(64, 64))
    assert c.infer(np.zeros((0, 3))).shape == (0, 8)
    for n in (1, 127, 129, 1000):
        pos = np.random.default_rng(n).uniform(-1, 1, (n, 3))
        np.testing.assert_allclose(c.infer(pos), c.infer(pos, precision=PRECISION_FP32), atol=FP16_VIS_TOL)


# ---------------------------------------------------------------------------
# geometry: G-buffer, factors, screen samples, targets
# ---------------------------------------------------------------------------
class TestGeometry:
    def test_gbuffer_bit_exact(self, boxes32, g_samp):
        cam = boxes32.camera.resized(40, 24)
        gb = make_gbuffer(boxes32, cam)
        np.testing.assert_array_equal(gb.flat("hit"), g_samp["gb_hit"])
        np.testing.assert_array_equal(gb.flat("position"), g_samp["gb_position"])
        np.testing.assert_array_equal(gb.flat("normal"), g_samp["gb_normal"])
        np.testing.assert_array_equal(gb.flat("albedo"), g_samp["gb_albedo"])
        np.testing.assert_array_equal(gb.flat("light_id"), g_samp["gb_light_id"])
        np.testing.assert_array_equal(gb.flat("depth"), g_samp["gb_depth"])
        np.testing.assert_array_equal(gb.flat("emissive"), g_samp["gb_emissive"])
        assert np.isinf(gb.flat("depth")[~gb.flat("hit")]).all()
        from paper_2506_05930_b200 import gbuffer_and_ctx
        gb2, ctx = gbuffer_and_ctx(boxes32, cam)             # (gb, ctx) as render.py:128-142
        assert gbuffer_and_ctx(boxes32, cam)[1] is ctx        # memoized per camera
        np.testing.assert_array_equal(gb2.flat("emissive"), g_samp["gb_emissive"])
        np.testing.assert_array_equal(ctx.normals, g_samp["gb_normal"])
        np.testing.assert_array_equal(ctx.albedos, g_samp["gb_albedo"])

    def test_point_gbuffer_and_factors(self, pbox8, g_samp):
        gb = make_gbuffer(pbox8)
        np.testing.assert_array_equal(gb.flat("position"), g_samp["pgb_position"])
        ctx = PixelCtx(pbox8, gb.flat("position"), gb.flat("normal"), gb.flat("albedo"), table_dtype=np.float64)
        np.testing.assert_allclose(ctx.factor_matrix(), g_samp["pgb_factor"], rtol=1e-12, atol=0)

    def test_rect_factors_and_lum(self, boxes32, g_samp):
        ctx = PixelCtx(boxes32, g_samp["gb_position"], g_samp["gb_normal"], g_samp["gb_albedo"],
                       table_dtype=np.float64)
        np.testing.assert_allclose(ctx.factor_matrix(), g_samp["nls_factor"], rtol=1e-10, atol=1e-300)
        np.testing.assert_allclose(ctx.lum_matrix(), g_samp["nls_lum"], rtol=1e-10, atol=1e-300)
        c32 = PixelCtx(boxes32, g_samp["gb_position"], g_samp["gb_normal"], g_samp["gb_albedo"])
        np.testing.assert_allclose(c32.lum_matrix(), g_samp["nls_lum"], rtol=1e-6, atol=1e-30)

    def test_screen_samples_bit_exact(self, boxes8, g_train):
        got = gen_screen_samples(boxes8, boxes8.camera, 256, R.stream(6))
        np.testing.assert_array_equal(got, g_train["screen_boxes8_256"])

    def test_screen_samples_all_miss(self):
        from paper_2506_05930_b200.scene import scene_from_dict as sfd
        s = sfd({"camera": {"position": [0, 0, 3], "look_at": [0, 0, 4], "up": [0, 1, 0], "fov_deg": 40.0,
                            "width": 16, "height": 16},
                 "materials": [{"albedo": [0.5, 0.5, 0.5]}],
                 "meshes": [{"material": 0, "triangles": [[[-1, 0, -1], [1, 0, -1], [1, 0, 1]]]}],
                 "lights": [{"type": "point", "position": [0, 2, 0], "intensity": [1, 1, 1]}]})
        assert gen_screen_samples(s, s.camera, 64, R.stream(5)).shape == (0, 3)

    def test_world_and_screen_samples_continue_a_used_stream(self, boxes8, g_scenes):
        """gen_world_samples / gen_screen_samples from a Generator that has already drawn:
        same points as numpy's own calls from there, and the stream ends where they leave it."""
        g, h = R.stream(3, "used-ws"), R.stream(3, "used-ws")
        g.random(7)
        h.random(7)
        np.testing.assert_array_equal(gen_world_samples(boxes8, 101, g),
                                      h.uniform(boxes8.aabb_min, boxes8.aabb_max, (101, 3)))
        np.testing.assert_array_equal(g.random(2), h.random(2))
        key, off = R.position(g)
        sa = O.SceneArrays.from_golden(g_scenes, "boxes8_")
        st = O.Stream(key=key, offset=off)
        want = O.screen_samples(sa, 300, st)
        np.testing.assert_array_equal(gen_screen_samples(boxes8, boxes8.camera, 300, g), want)
        np.testing.assert_array_equal(g.random(3), O.uniform_at(key, st.offset + np.arange(3)))

    def test_c1_train_batch_bit_exact(self, pbox8, g_train):
        key = (0, 0, 0)
        world = gen_world_samples(pbox8, 4096, R.stream(*key, R.WORLD_SAMPLES))
        screen = gen_screen_samples(pbox8, pbox8.camera, 4096, R.stream(*key, R.SCREEN_SAMPLES))
        pos = np.concatenate([world, screen])
        np.testing.assert_array_equal(pos, g_train["c1_pos"])
        tgt = compute_visibility_targets(pos, pbox8, R.stream(*key, R.TARGETS))
        np.testing.assert_array_equal(tgt.astype(np.uint8), g_train["c1_tgt"])

    @pytest.mark.parametrize("shards,unsorted,anyhit", [(1, False, "auto"), (2, False, "auto"), (3, False, "auto"),
                                                        (1, True, "auto"), (2, True, "auto"), (1, False, "bvh"),
                                                        (1, True, "bvh"), (1, False, "bf")])
    def test_boxes32_device_batch_bit_exact(self, g_train, shards, unsorted, anyhit, monkeypatch):
        """Batch positions and shadow-ray targets (Morton-bucketed warps, and the plain
        row-per-warp kernel; plane-culled any-hit and the packet BVH traversal) are
        bit-identical to the reference, also per shard."""
        from paper_2506_05930_b200.training import BatchBuffers, gen_batch_device
        if unsorted:
            monkeypatch.setenv("NVC_TARGETS_UNSORTED", "1")
        monkeypatch.setenv("NVC_ANYHIT", anyhit)
        boxes32 = scene_from_dict(boxes_scene(32))       # fresh DeviceScene picks up NVC_ANYHIT
        pos_all, tgt_all = [], []
        for sh in range(shards):
            bufs = BatchBuffers(2048, 2048, 32, DEV, shards)
            gen_batch_device(boxes32, boxes32.camera, bufs, 0, 3, 0, sh, shards)
            b = int(bufs.n_rows.item())
            lo, hi = b * sh // shards, b * (sh + 1) // shards
            pos_all.append(bufs.pos[:b].cpu().numpy())
            tgt_all.append(bufs.tgt[:hi - lo].cpu().numpy())
        np.testing.assert_array_equal(pos_all[0], g_train["b32_pos"])
        np.testing.assert_array_equal(np.concatenate(tgt_all).astype(np.uint8), g_train["b32_tgt"])


# ---------------------------------------------------------------------------
# any-hit strategies + shading pass 5 (render.py:220-246)
# ---------------------------------------------------------------------------
def _scene_with(name_fn, anyhit, monkeypatch):
    monkeypatch.setenv("NVC_ANYHIT", anyhit)
    return scene_from_dict(name_fn())


def _visibility(scene, x, y):
    from paper_2506_05930_b200.scene import device_scene
    ds = device_scene(scene, DEV)
    xt, yt = (torch.from_numpy(np.ascontiguousarray(a)).to(DEV) for a in (x, y))
    vis = torch.empty(x.shape[0], dtype=torch.float32, device=DEV)
    _lib.call("nvc_visibility", ds.struct, xt.data_ptr(), yt.data_ptr(), x.shape[0], vis.data_ptr(),
              _lib.stream_ptr())
    return vis.cpu().numpy()


class TestShade:
    @pytest.mark.parametrize("anyhit", ["auto", "bf", "bvh"])
    def test_golden_boxes32(self, g_shade, anyhit, monkeypatch):
        from paper_2506_05930_b200.render import shade_batch
        s = _scene_with(lambda: boxes_scene(32), anyhit, monkeypatch)
        z = g_shade
        rgb = shade_batch(s, z["b32_position"], z["b32_normal"], z["b32_albedo"], z["b32_ids"], z["b32_pts"],
                          z["b32_W"])
        np.testing.assert_array_equal(rgb, z["b32_rgb"])

    def test_golden_point_lights_and_nls_chain(self, pbox8, boxes32, g_samp, g_shade):
        from paper_2506_05930_b200.render import shade_batch, shade_pixel
        from paper_2506_05930_b200.sampling import ShadingPoint
        z = g_shade
        rgb = shade_batch(pbox8, g_samp["pgb_position"], g_samp["pgb_normal"], g_samp["pgb_albedo"], z["p8_ids"],
                          z["p8_pts"], z["p8_W"])
        np.testing.assert_array_equal(rgb, z["p8_rgb"])
        rgb = shade_batch(boxes32, g_samp["gb_position"], g_samp["gb_normal"], g_samp["gb_albedo"],
                          g_samp["nls_ids"], g_samp["nls_pts"], g_samp["nls_W"])
        np.testing.assert_array_equal(rgb, z["nls_rgb"])
        i = int(np.argmax(np.abs(z["nls_rgb"]).sum(axis=1)))
        sp = ShadingPoint(g_samp["gb_position"][i], g_samp["gb_normal"][i], g_samp["gb_albedo"][i])
        one = shade_pixel(sp, (int(g_samp["nls_ids"][i]), g_samp["nls_pts"][i], float(g_samp["nls_W"][i])), boxes32)
        np.testing.assert_array_equal(one, z["nls_rgb"][i])
        with pytest.raises(ValueError):
            shade_pixel(sp, (0, g_samp["nls_pts"][i], -1.0), boxes32)

    @pytest.mark.parametrize("anyhit", ["auto", "bf", "bvh"])
    def test_large_random_vs_oracle(self, g_scenes, anyhit, monkeypatch):
        """200k G-buffer rows (320x...) with random (id, point, W), ids in [-1, K]."""
        from paper_2506_05930_b200.render import gbuffer_device, shade_device
        s = _scene_with(lambda: boxes_scene(32), anyhit, monkeypatch)
        cam = s.camera.resized(480, 416)
        pos, nrm, alb, _, _ = gbuffer_device(s, cam, device=DEV)
        n = pos.shape[0]
        g = np.random.default_rng(7)
        ids = g.integers(-1, 33, size=n)                 # K = 32 -> id 32 is out of range: row is 0
        u = g.random((n, 2))
        o = O.SceneArrays.from_golden(g_scenes, "boxes32_")
        pts = o.light_points(np.minimum(np.maximum(ids, 0), 31), u)
        big_w = g.random(n) * 30.0 * (g.random(n) < 0.95)
        rgb = shade_device(s, pos, nrm, alb, torch.from_numpy(ids).to(DEV), torch.from_numpy(pts).to(DEV),
                           torch.from_numpy(big_w).to(DEV)).cpu().numpy()
        ids_o = np.where(ids >= 32, -1, ids)
        want = O.shade(o, pos.cpu().numpy(), nrm.cpu().numpy(), alb.cpu().numpy(), ids_o, pts, big_w)
        np.testing.assert_array_equal(rgb, want)
        assert (rgb != 0).any(axis=1).sum() > n // 10

    def test_warp_culled_targets_equal_bvh_over_frames(self, monkeypatch):
        """Shadow-ray targets of 8 full C2 batches (2 M rays): warp-level + per-lane
        culling (default), per-lane only, and the packet BVH traversal agree bitwise."""
        from paper_2506_05930_b200.training import BatchBuffers, gen_batch_device
        got = {}
        for mode in ("auto", "bf", "bvh"):
            s = _scene_with(lambda: boxes_scene(32), mode, monkeypatch)
            outs = []
            for f in range(8):
                bufs = BatchBuffers(4096, 4096, 32, DEV, 1)
                gen_batch_device(s, s.camera.resized(1920, 1080), bufs, 0, f, 0, 0, 1)
                outs.append(bufs.tgt.cpu().numpy().copy())
            got[mode] = np.stack(outs)
        np.testing.assert_array_equal(got["auto"], got["bvh"])
        np.testing.assert_array_equal(got["bf"], got["bvh"])
        assert 0.05 < got["bvh"].mean() < 0.95

    @pytest.mark.parametrize("scene_fn", [lambda: boxes_scene(32), lambda: rooms_scene(32)])
    def test_warp_shaft_filter_grazing_rows(self, scene_fn, monkeypatch):
        """The warp filter's shaft / plane-side / crossing-box culling against rows
        placed ON scene triangles (and 1e-12 .. 1e-3 off them, on both sides), so many
        of the 32 shadow rays of a row graze a plane or start inside one: targets
        agree bitwise with per-lane culling and with the BVH traversal."""
        from paper_2506_05930_b200.training import compute_visibility_targets
        s0 = scene_from_dict(scene_fn())
        g = np.random.default_rng(11)
        tri = g.integers(0, s0.triangles_v0.shape[0], 6000)
        u = g.random((6000, 2))
        flip = u.sum(1) > 1.0
        u[flip] = 1.0 - u[flip]
        v0, v1, v2 = s0.triangles_v0[tri], s0.triangles_v1[tri], s0.triangles_v2[tri]
        p = v0 + u[:, :1] * (v1 - v0) + u[:, 1:] * (v2 - v0)
        nrm = np.cross(v1 - v0, v2 - v0)
        nrm /= np.maximum(np.linalg.norm(nrm, axis=1, keepdims=True), 1e-300)
        off = np.array([0.0, 1e-12, -1e-12, 1e-9, -1e-9, 1e-6, -1e-6, 1e-3, -1e-3, 0.0])[g.integers(0, 10, 6000)]
        pos = np.concatenate([p + off[:, None] * nrm, g.uniform(s0.aabb_min, s0.aabb_max, (2192, 3))])
        got = {}
        for mode in ("auto", "bf", "bvh"):
            s = _scene_with(scene_fn, mode, monkeypatch)
            got[mode] = compute_visibility_targets(pos, s, R.Stream(5, 0, 0, "grazing"))
        np.testing.assert_array_equal(got["auto"], got["bvh"])
        np.testing.assert_array_equal(got["bf"], got["bvh"])
        assert 0.05 < got["bvh"].mean() < 0.95

    @pytest.mark.parametrize("scene_fn", [lambda: boxes_scene(32), lambda: boxes_point_scene(8)])
    def test_plane_culling_equals_bvh_traversal(self, scene_fn, monkeypatch):
        """1M random segments inside (and beyond) the scene box, plus segments between
        surface points: the plane-culled any-hit and the BVH traversal agree bitwise."""
        bf = _scene_with(scene_fn, "bf", monkeypatch)
        bvh = _scene_with(scene_fn, "bvh", monkeypatch)
        g = np.random.default_rng(3)
        lo, hi = bf.aabb_min - 0.5, bf.aabb_max + 0.5
        x = g.uniform(lo, hi, (1 << 20, 3))
        y = g.uniform(lo, hi, (1 << 20, 3))
        y[::7] = x[::7] + 1e-5 * g.standard_normal((y[::7].shape[0], 3))     # short / degenerate segments
        a = _visibility(bf, x, y)
        b = _visibility(bvh, x, y)
        np.testing.assert_array_equal(a, b)
        assert 0.05 < a.mean() < 0.95


# ---------------------------------------------------------------------------
# light selection: NLS / Neural DI
# ---------------------------------------------------------------------------
class FixedCache:
    mode = MODE_LIGHTS

    def __init__(self, vis):
        self.vis = np.asarray(vis, np.float32)
        self.output_dim = self.vis.shape[1]

    def infer(self, positions):
        return self.vis[: positions.shape[0]]


class TestSampling:
    def test_nls_bit_exact_vs_reference(self, boxes32, g_samp):
        ctx = PixelCtx(boxes32, g_samp["gb_position"], g_samp["gb_normal"], g_samp["gb_albedo"],
                       factors=g_samp["nls_factor"], table_dtype=np.float64)
        ctx._lum = torch.from_numpy(np.ascontiguousarray(g_samp["nls_lum"].T)).to(DEV)
        ids, pts, big_w = nls_sample_batch(ctx, FixedCache(g_samp["nls_vis"]), R.stream(0, 7, "light-select"))
        np.testing.assert_array_equal(ids, g_samp["nls_ids"])
        np.testing.assert_array_equal(pts, g_samp["nls_pts"])
        np.testing.assert_array_equal(big_w, g_samp["nls_W"])
        ids, _, big_w = nls_sample_batch(ctx, FixedCache(g_samp["nls_vis"]), R.stream(0, 7, "light-select"), 0.0)
        np.testing.assert_array_equal(ids, g_samp["nls_ids_biased"])
        np.testing.assert_array_equal(big_w, g_samp["nls_W_biased"])

    @pytest.mark.parametrize("variant", ["default", "NVC_WRS_FORWARD", "NVC_ENC_F32", "NVC_MLP_QUADS"])
    def test_fused_nls_equals_oracle_on_same_visibility(self, boxes32, g_samp, g_scenes, variant, monkeypatch):
        """The query's WRS is bit-exact given its own (fp16-MLP) visibilities -- for the default
        kernels and each alternative (generic reservoir, scalar encoder, SS-mode MLP)."""
        if variant != "default":
            monkeypatch.setenv(variant, "1")
        c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(boxes32, 16, 1 << 19), hidden_dims=(64, 64, 64))
        c.grid_params = (np.random.default_rng(0).standard_normal(c.grid_params.shape) * 0.5).astype(np.float32)
        ctx = PixelCtx(boxes32, g_samp["gb_position"], g_samp["gb_normal"], g_samp["gb_albedo"])
        vis16 = c.infer(g_samp["gb_position"], precision=PRECISION_FP16)
        lum = ctx.lum_matrix()          # f32 table widened to f64, as the kernel does
        sc = O.SceneArrays.from_golden(g_scenes, "boxes32_")
        key = R.stream_key(0, 9, "light-select")
        for offset in (0, 1, 2, 3):   # 0: block-aligned group kernel; others: per-light kernel
            oi, op, ow = O.nls_sample(sc, vis16, lum, key, offset=offset)
            ids, pts, big_w = nls_sample_batch(ctx, c, R.Stream(key=key, offset=offset))
            np.testing.assert_array_equal(ids, oi)
            np.testing.assert_array_equal(pts, op)
            np.testing.assert_array_equal(big_w, ow)
            assert (ids >= 0).sum() > 100

    @pytest.mark.parametrize("k,hidden", [(64, (64, 64, 64)), (128, (128, 128, 128))])
    def test_wide_k_nls_equals_oracle(self, k, hidden, monkeypatch):
        """K = 64 / 128 (rooms scenes, C4's 3x128 MLP): the grouped reservoir over 2 / 4
        mask words (block-aligned offset) and the generic one (offset 1) are bit-exact."""
        from paper_2506_05930_b200.render import gbuffer_device
        from paper_2506_05930_b200.scenes import rooms_scene
        s = scene_from_dict(rooms_scene(k))
        cam = s.camera.resized(64, 40)
        pos, nrm, alb, _, _ = gbuffer_device(s, cam)
        ctx = PixelCtx(s, pos, nrm, alb)
        c = VisibilityCache(MODE_LIGHTS, k, grid_cfg(s, 16, 1 << 19), hidden_dims=hidden)
        c.grid_params = (np.random.default_rng(2).standard_normal(c.grid_params.shape) * 0.5).astype(np.float32)
        vis16 = c.infer(pos.cpu().numpy(), precision=PRECISION_FP16)
        sc = O.SceneArrays(s.triangles_v0, s.triangles_v1, s.triangles_v2, s.tri_material, s.tri_light, s.lt_kind,
                           s.lt_verts, s.lt_normal, s.lt_radiance, s.mat_albedo, np.zeros(12))
        lum = ctx.lum_matrix()
        assert (lum != 0).any(axis=1).sum() > 100 and (lum == 0).any()
        key = R.stream_key(0, 3, "light-select")
        for offset in (0, 1):
            oi, op, ow = O.nls_sample(sc, vis16, lum, key, offset=offset)
            ids, pts, big_w = nls_sample_batch(ctx, c, R.Stream(key=key, offset=offset))
            np.testing.assert_array_equal(ids, oi)
            np.testing.assert_array_equal(pts, op)
            np.testing.assert_array_equal(big_w, ow)
            assert (ids >= 32).any()

    @pytest.mark.parametrize("grid", ["3", "7"])
    def test_fused_pipeline_many_tiles_per_cta(self, boxes32, g_scenes, monkeypatch, grid):
        """Few CTAs -> every CTA cycles its A0 / TMEM / lum stages many times."""
        from paper_2506_05930_b200.render import gbuffer_device
        cam = boxes32.camera.resized(96, 54)
        pos, nrm, alb, _, _ = gbuffer_device(boxes32, cam)
        ctx = PixelCtx(boxes32, pos, nrm, alb)
        c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(boxes32, 16, 1 << 19), hidden_dims=(64, 64, 64))
        c.grid_params = (np.random.default_rng(1).standard_normal(c.grid_params.shape) * 0.5).astype(np.float32)
        vis16 = c.infer(pos.cpu().numpy(), precision=PRECISION_FP16)
        sc = O.SceneArrays.from_golden(g_scenes, "boxes32_")
        key = R.stream_key(0, 12, "light-select")
        oi, op, ow = O.nls_sample(sc, vis16, ctx.lum_matrix(), key)
        monkeypatch.setenv("NVC_QUERY_GRID", grid)
        np.testing.assert_array_equal(c.infer(pos.cpu().numpy(), precision=PRECISION_FP16), vis16)
        ids, pts, big_w = nls_sample_batch(ctx, c, R.Stream(key=key))
        np.testing.assert_array_equal(ids, oi)
        np.testing.assert_array_equal(pts, op)
        np.testing.assert_array_equal(big_w, ow)
        rgb = neural_di_batch(ctx, c)
        f = ctx.factor_matrix()
        want = ((vis16.astype(np.float64) * f) @ boxes32.lt_radiance) * alb.cpu().numpy() / np.pi
        np.testing.assert_allclose(rgb, want, rtol=1e-9, atol=1e-12)

    def test_stage_profiling_hook(self, boxes32):
        """nvc_profile_stages / nvc_profile_stage_ms time the three query kernels."""
        import ctypes
        from paper_2506_05930_b200 import _lib
        from paper_2506_05930_b200.render import gbuffer_device
        pos, nrm, alb, _, _ = gbuffer_device(boxes32, boxes32.camera.resized(64, 32))
        ctx = PixelCtx(boxes32, pos, nrm, alb)
        c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(boxes32, 16, 1 << 19), hidden_dims=(64, 64, 64))
        _lib.call("nvc_profile_stages", 1)
        nls_sample_batch(ctx, c, R.Stream(key=R.stream_key(0, 1, "light-select")))
        _lib.call("nvc_profile_stages", 0)
        ms = (ctypes.c_float * 3)()
        _lib.call("nvc_profile_stage_ms", ctypes.addressof(ms))
        assert all(0.0 < x < 1000.0 for x in ms)

    def test_select_on_side_stream_matches_inline(self, boxes32):
        """nvc_query_front + nvc_nls_select on another stream == nvc_nls_sample."""
        from paper_2506_05930_b200.render import gbuffer_device
        from paper_2506_05930_b200.sampling import nls_sample_device
        pos, nrm, alb, _, _ = gbuffer_device(boxes32, boxes32.camera.resized(96, 54))
        ctx = PixelCtx(boxes32, pos, nrm, alb)
        c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(boxes32, 16, 1 << 19), hidden_dims=(64, 64, 64))
        key = R.stream_key(0, 4, "light-select")
        want = [t.clone() for t in nls_sample_device(ctx, c, key)]
        side = torch.cuda.Stream()
        got = nls_sample_device(ctx, c, key, select_stream=side)
        torch.cuda.current_stream().wait_event(c.select_done)
        for a, b in zip(want, got):
            assert torch.equal(a, b)
        # back-to-back frames: the query workspaces alternate, so frame f+1's encoder
        # and MLP run while frame f's selection may still read its workspace
        keys = [R.stream_key(0, f, "light-select") for f in range(5)]
        want = [[t.clone() for t in nls_sample_device(ctx, c, k)] for k in keys]
        got = [nls_sample_device(ctx, c, k, select_stream=side) for k in keys]
        torch.cuda.current_stream().wait_event(c.select_done)
        for w, g in zip(want, got):
            for a, b in zip(w, g):
                assert torch.equal(a, b)

    def test_tile_sharded_nls_matches_whole_frame(self, boxes32, g_samp):
        from paper_2506_05930_b200.sampling import nls_sample_device
        c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(boxes32, 16, 1 << 19), hidden_dims=(64, 64, 64))
        pos, nrm, alb = g_samp["gb_position"], g_samp["gb_normal"], g_samp["gb_albedo"]
        key = R.stream_key(0, 11, "light-select")
        whole = PixelCtx(boxes32, pos, nrm, alb)
        wi, wp, ww = (t.cpu().numpy() for t in nls_sample_device(whole, c, key))
        cuts = [0, 333, 640, pos.shape[0]]
        for a, b in zip(cuts[:-1], cuts[1:]):
            part = PixelCtx(boxes32, pos[a:b], nrm[a:b], alb[a:b])
            si, sp, sw = (t.cpu().numpy() for t in nls_sample_device(part, c, key, p_first=a,
                                                                     p_total=pos.shape[0]))
            np.testing.assert_array_equal(si, wi[a:b])
            np.testing.assert_array_equal(sp, wp[a:b])
            np.testing.assert_array_equal(sw, ww[a:b])

    def test_neural_di(self, boxes32, g_samp):
        ctx = PixelCtx(boxes32, g_samp["gb_position"], g_samp["gb_normal"], g_samp["gb_albedo"],
                       table_dtype=np.float64)
        got = neural_di_batch(ctx, FixedCache(g_samp["nls_vis"]))
        np.testing.assert_allclose(got, g_samp["ndi_rgb"], rtol=1e-9, atol=1e-12)
        c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(boxes32, 16, 1 << 19), hidden_dims=(64, 64, 64))
        vis16 = c.infer(g_samp["gb_position"])
        want = ((vis16.astype(np.float64) * ctx.factor_matrix()) @ boxes32.lt_radiance) * g_samp["gb_albedo"] / np.pi
        np.testing.assert_allclose(neural_di_batch(ctx, c), want, rtol=1e-9, atol=1e-12)

    def test_neural_di_f32_table_kernel(self, boxes32, g_samp):
        """The f32-factor-table Neural DI kernel (k_ndi32: the warp walks the union of
        its pixels' nonzero lights, factors in registers) equals the per-pixel
        ascending-light FP64 sum op for op: sum_k (v_k f_k) L_e[k], then * albedo / pi."""
        from paper_2506_05930_b200.render import gbuffer_device
        pos, nrm, alb, _, _ = gbuffer_device(boxes32, boxes32.camera.resized(320, 180))
        ctx = PixelCtx(boxes32, pos, nrm, alb, table_dtype=np.float32)
        c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(boxes32, 16, 1 << 19), hidden_dims=(64, 64, 64))
        c.grid_params = (np.random.default_rng(4).standard_normal(c.grid_params.shape) * 0.3).astype(np.float32)
        got = neural_di_batch(ctx, c)
        vis = c.infer(pos.cpu().numpy()).astype(np.float64)
        fac = ctx.factor_matrix().astype(np.float64)
        le = boxes32.lt_radiance
        rgb = np.zeros((vis.shape[0], 3))
        for k in range(vis.shape[1]):
            wk = vis[:, k] * fac[:, k]
            rgb = rgb + wk[:, None] * le[k][None, :]
        want = rgb * alb.cpu().numpy() / np.pi
        np.testing.assert_array_equal(got, want)
        assert (got != 0).any(axis=1).mean() > 0.5


# ---------------------------------------------------------------------------
# training: Adam, one step, loss curve, determinism, shard equivalence
# ---------------------------------------------------------------------------
class TestTraining:
    def _c1(self, pbox8, seed=0):
        return VisibilityCache(MODE_LIGHTS, 8, grid_cfg(pbox8, 8, 1 << 14), seed=seed, hidden_dims=(64, 64))

    @pytest.mark.parametrize("kernel", ["dense2", "bulk4", "flat", "no_side_stream"])
    def test_adam_bit_exact_given_grads(self, pbox8, kernel, monkeypatch):
        env = {"flat": "NVC_ADAM_FLAT", "bulk4": "NVC_ADAM_BULK4", "no_side_stream": "NVC_NO_SIDE_STREAM"}
        if kernel in env:
            monkeypatch.setenv(env[kernel], "1")
        c = self._c1(pbox8)
        c.set_compact(False)          # feed arbitrary dense gradients
        p0 = c.params.cpu().numpy().copy()
        g = np.random.default_rng(5)
        st = O.Adam(p0.size)
        p = p0.copy()
        for t in range(3):
            gd = (g.standard_normal(p0.size) * 10.0 ** g.integers(-7, 0, p0.size))
            # fixed point: 2^-48 for the hash table, 2^-58 for the MLP (common.cuh)
            scale = np.where(np.arange(p0.size) < c.grid_cfg.param_count, 2.0 ** 48, 2.0 ** 58)
            fx = np.rint(gd * scale).astype(np.int64)
            gf = (fx.astype(np.float64) / scale).astype(np.float32)   # what the kernel reads
            c.grad_fx.copy_(torch.from_numpy(fx))
            lr = 0.05 - 0.001 * t
            c.step = 0
            c.train_cfg.lr_start = lr
            c.train_cfg.lr_end = min(lr, c.train_cfg.lr_end)
            c.apply_adam()
            st.step(p, gf, lr)
            np.testing.assert_array_equal(c.params.cpu().numpy(), p)
        np.testing.assert_array_equal(c.adam_m.cpu().numpy(), st.m)
        np.testing.assert_array_equal(c.adam_v.cpu().numpy(), st.v)
        assert not c.grad_fx.any()
        gcfg = c.grid_cfg
        t2 = c.table_h.cpu().numpy().reshape(gcfg.levels, gcfg.table_size, 2, gcfg.features_per_level)
        tab = p[:gcfg.param_count].astype(np.float16).reshape(gcfg.levels, gcfg.table_size, gcfg.features_per_level)
        np.testing.assert_array_equal(t2[:, :, 0], tab)                       # own slot
        np.testing.assert_array_equal(t2[:, :, 1], np.roll(tab, -1, axis=1))  # x-neighbour (mod T)

    @pytest.mark.parametrize("compact", [True, False])
    def test_bulk_and_flat_adam_agree_and_consume_grads(self, pbox8, g_train, monkeypatch, compact):
        a, b = self._c1(pbox8), self._c1(pbox8)
        pt = torch.from_numpy(g_train["c1_pos"]).to(DEV)
        tt = torch.from_numpy(g_train["c1_tgt"].astype(np.float32)).to(DEV)
        for c, flat in ((a, False), (b, True)):
            c.set_compact(compact)
            if flat:
                monkeypatch.setenv("NVC_ADAM_FLAT", "1")
            c.accumulate_grads(pt, tt)
            acc = c.grad_c if compact else c.grad_fx
            assert acc.any()
            c.apply_adam()
            assert not acc.any()                # the accumulator is consumed (zeroed) by Adam
        np.testing.assert_array_equal(a.params.cpu().numpy(), b.params.cpu().numpy())
        np.testing.assert_array_equal(a.table_h.cpu().numpy(), b.table_h.cpu().numpy())

    def test_first_step_vs_reference(self, pbox8, g_train):
        c = self._c1(pbox8)
        loss = c.train_step(g_train["c1_pos"], g_train["c1_tgt"].astype(np.float32))
        assert loss == pytest.approx(float(g_train["c1_step0_loss"]), rel=1e-6)
        np.testing.assert_allclose(c.net_params.weights[0], g_train["c1_step0_w0"], atol=2e-6)

    @pytest.mark.parametrize("kind", ["binary", "fractional"])
    def test_masked_train_step_vs_oracle(self, pbox8, g_train, kind):
        """train_step(positions, targets, mask): masked loss and gradients (mlp.py:143-168)
        against the oracle on the C1 batch."""
        pos, tgt = g_train["c1_pos"], g_train["c1_tgt"].astype(np.float32)
        g = np.random.default_rng(8)
        mask = (g.random(tgt.shape) < 0.7).astype(np.float32) if kind == "binary" else \
            g.random(tgt.shape).astype(np.float32)
        c = self._c1(pbox8)
        oc = O.Cache(O.Grid(levels=8, features_per_level=2, table_size=1 << 14, aabb_min=pbox8.aabb_min,
                            aabb_max=pbox8.aabb_max), 8, hidden=(64, 64), seed=0)
        loss = c.train_step(pos, tgt, mask)
        oloss = oc.train_step(pos, tgt, mask)
        assert loss == pytest.approx(oloss, rel=1e-6)
        np.testing.assert_allclose(c.net_params.weights[0], oc.ws[0], atol=2e-6)

    def test_loss_curve_vs_reference(self, pbox8, g_train):
        c = self._c1(pbox8)
        want = g_train["c1_loss_f32"]
        got = [train_frame(pbox8, pbox8.camera, c, TrainFrameConfig(), frame=f) for f in range(len(want))]
        np.testing.assert_allclose(got, want, rtol=1e-2)      # FP32 vs reference FP32; SURVEY §8(c) band
        ref64 = g_train["c1_loss_f64"]
        assert np.max(np.abs(np.array(got) - ref64) / ref64) < 1e-2

    def test_tensor_core_training_step(self, pbox8, g_train, monkeypatch):
        """tcgen05 training step (split bf16 operands, fp32 TMEM accumulators):
        deterministic, first-step loss and weights at the fp32 path's tolerances,
        the C1 loss curve within the same 1e-2 band as the fp32 SIMT step."""
        monkeypatch.setenv("NVC_TRAIN_TC", "1")
        c = self._c1(pbox8)
        loss = c.train_step(g_train["c1_pos"], g_train["c1_tgt"].astype(np.float32))
        assert loss == pytest.approx(float(g_train["c1_step0_loss"]), rel=1e-6)
        np.testing.assert_allclose(c.net_params.weights[0], g_train["c1_step0_w0"], atol=2e-6)
        c = self._c1(pbox8)
        want = g_train["c1_loss_f32"]
        got = [train_frame(pbox8, pbox8.camera, c, TrainFrameConfig(), frame=f) for f in range(len(want))]
        np.testing.assert_allclose(got, want, rtol=1e-2)
        c2 = self._c1(pbox8)
        again = [train_frame(pbox8, pbox8.camera, c2, TrainFrameConfig(), frame=f) for f in range(len(want))]
        assert got == again

    def test_tensor_core_gradients_match_fp32(self, boxes32, g_train, monkeypatch):
        """The tcgen05 step's gradients against the fp32 SIMT step's on a C2-shaped
        batch: MLP gradients within 1e-3 of each block's largest (w0 is the worst,
        ~6e-4: the init-scale features), hash-grid gradients within 1e-4 relative
        for 99 % of the touched entries (the rest: leaky-ReLU kinks, z ~ 0)."""
        pos = torch.from_numpy(g_train["b32_pos"]).to(DEV)
        tgt = torch.from_numpy(g_train["b32_tgt"].astype(np.float32)).to(DEV)
        out = []
        for tc in (False, True):
            if tc:
                monkeypatch.setenv("NVC_TRAIN_TC", "1")
            c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(boxes32, 16, 1 << 19), seed=0, hidden_dims=(64, 64, 64))
            c.set_compact(False)
            c.accumulate_grads(pos, tgt)
            out.append(c.grad_fx.double().cpu().numpy() * 2.0 ** -48)
        a, b = out
        n = c.grid_cfg.param_count
        for (wo, bo), (fo, fi) in zip(c._layer_offs, c.net_cfg.layer_dims):
            for sl in (slice(wo, wo + fo * fi), slice(bo, bo + fo)):
                assert np.abs(a[sl] - b[sl]).max() <= 1e-3 * np.abs(a[sl]).max()
        live = np.abs(a[:n]) > 1e-3 * np.abs(a[:n]).max()
        rel = np.abs(a[:n][live] - b[:n][live]) / np.abs(a[:n][live])
        assert np.quantile(rel, 0.99) < 1e-4

    def test_bitwise_deterministic_trajectory(self, pbox8):
        def run():
            c = self._c1(pbox8, seed=5)
            cfg = TrainFrameConfig(n_world=512, n_screen=512, seed=5)
            return [train_frame(pbox8, pbox8.camera, c, cfg, frame=f) for f in range(3)], c.params.cpu().numpy()
        la, pa = run()
        lb, pb = run()
        assert la == lb
        np.testing.assert_array_equal(pa, pb)

    def test_compact_exchange_equals_dense_allreduce(self, pbox8, g_train):
        """GradExchange: pack -> sum over shards -> unpack == full-batch grad_fx, bit for bit."""
        pos = torch.from_numpy(g_train["c1_pos"]).to(DEV)
        tgt = torch.from_numpy(g_train["c1_tgt"].astype(np.float32)).to(DEV)
        b = pos.shape[0]
        full = self._c1(pbox8)
        full.set_compact(False)
        full.accumulate_grads(pos, tgt)
        shards = [self._c1(pbox8) for _ in range(3)]
        for sh, c in enumerate(shards):
            c.set_compact(False)
            lo, hi = b * sh // 3, b * (sh + 1) // 3
            c.accumulate_grads(pos, tgt[lo:hi].contiguous(), b_max=b, shard=sh, n_shards=3)
            ex = c.exchange(b)
            ex.index(pos)
            ex.pack()
        total = sum(c.exchange(b).buf for c in shards)
        assert 0 < int(shards[0].exchange(b).count.item()) <= shards[0].exchange(b).max_entries
        ex0 = shards[0].exchange(b)
        ex0.buf.copy_(total)
        ex0.unpack()
        gc = full.grid_cfg.param_count
        np.testing.assert_array_equal(full.grad_fx[:gc].cpu().numpy(), shards[0].grad_fx[:gc].cpu().numpy())
        np.testing.assert_allclose(full.grad_fx[gc:].double().cpu().numpy(),
                                   shards[0].grad_fx[gc:].double().cpu().numpy(), rtol=1e-5, atol=2.0 ** 58 * 1e-9)

    def test_wide_split_train_equals_fused_kernel(self, boxes32, monkeypatch):
        """C4 widths (3x128 hidden, 128 outputs): the split step with W read from L1/L2
        (k_train3<true>) and the single fused fp32 kernel (k_mlp<true>) produce
        bit-identical parameters after three steps (same arithmetic and row partition)."""
        g = np.random.default_rng(5)
        pos = torch.from_numpy(g.uniform(boxes32.aabb_min, boxes32.aabb_max, (3000, 3))).to(DEV)
        tgt = torch.from_numpy((g.random((3000, 128)) < 0.5).astype(np.float32)).to(DEV)

        def run(fused):
            if fused:
                monkeypatch.setenv("NVC_TRAIN_FUSED", "1")
            else:
                monkeypatch.delenv("NVC_TRAIN_FUSED", raising=False)
            c = VisibilityCache(MODE_LIGHTS, 128, grid_cfg(boxes32, 16, 1 << 19), seed=1,
                                hidden_dims=(128, 128, 128))
            losses = [c.train_step(pos, tgt) for _ in range(3)]
            return c.params.cpu().numpy(), losses

        (pa, la), (pb, lb) = run(False), run(True)
        np.testing.assert_array_equal(pa, pb)
        assert la == lb

    def test_compact_gradients_match_dense(self, pbox8, g_train):
        """Compact gradient slots train exactly like the dense accumulator (same arithmetic,
        same integer sums): identical parameters after three steps, whole-batch and with two
        row shards whose compact buffers are summed as the allreduce would."""
        pos = torch.from_numpy(g_train["c1_pos"]).to(DEV)
        tgt = torch.from_numpy(g_train["c1_tgt"].astype(np.float32)).to(DEV)
        b = pos.shape[0]

        def run(compact, shards):
            ranks = [self._c1(pbox8) for _ in range(shards)]
            for c in ranks:
                c.set_compact(compact)
            for step in range(3):
                for r, c in enumerate(ranks):
                    lo, hi = b * r // shards, b * (r + 1) // shards
                    c.accumulate_grads(pos, tgt[lo:hi].contiguous(), b_max=b, shard=r, n_shards=shards)
                acc = [c.grad_c if compact else c.grad_fx for c in ranks]
                total = sum(acc)
                for t in acc:
                    t.copy_(total)
                for c in ranks:
                    c.apply_adam()
            return ranks[0].params.cpu().numpy()

        for shards in (1, 2):
            np.testing.assert_array_equal(run(False, shards), run(True, shards))

    def test_batch_pipeline_matches_inline_generation(self, pbox8):
        """Batches prefetched one frame ahead on a side stream train bit-identically."""
        from paper_2506_05930_b200.training import BatchPipeline, train_frame_device
        cfg = TrainFrameConfig(n_world=512, n_screen=512, seed=3)
        a, b = self._c1(pbox8, seed=3), self._c1(pbox8, seed=3)
        pipe = BatchPipeline(pbox8, pbox8.camera, cfg, 8, DEV)
        la, lb = [], []
        for f in range(4):
            la.append(float(train_frame_device(pbox8, pbox8.camera, a, cfg, frame=f)[0]))
            lb.append(float(train_frame_device(pbox8, pbox8.camera, b, cfg, frame=f, pipeline=pipe)[0]))
        assert la == lb
        np.testing.assert_array_equal(a.params.cpu().numpy(), b.params.cpu().numpy())

    def test_batch_pipeline_builds_the_exchange_index(self, pbox8):
        """With data parallelism the pipeline lists the batch's table entries on its side stream:
        identical to building the list inline from the same positions."""
        from paper_2506_05930_b200 import GradExchange
        from paper_2506_05930_b200.training import BatchPipeline
        cfg = TrainFrameConfig(n_world=512, n_screen=512, seed=3)
        c = self._c1(pbox8, seed=3)
        pipe = BatchPipeline(pbox8, pbox8.camera, cfg, 8, DEV, shard=1, n_shards=2, cache=c)
        for f in range(3):
            bufs = pipe.take(f)
            ex = pipe.exchange_for(bufs)
            ref = GradExchange(c, cfg.n_world + cfg.n_screen)
            ref.index(bufs.pos, bufs.n_rows)
            n = int(ref.count.item())
            assert n > 0 and int(ex.count.item()) == n
            assert torch.equal(ex.idx[:n], ref.idx[:n])
            pipe.release(bufs, f)

    def test_reference_determinism_config_loss(self, g_train):
        """levels=4, T=2^10, 64+64 batch, seed 5 (test_mlp.py:205-224): loss within 1e-4."""
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
        c = VisibilityCache(MODE_LIGHTS, 1, HashGridConfig(levels=4, table_size=1 << 10, aabb_min=ps.aabb_min,
                                                           aabb_max=ps.aabb_max), seed=5)
        cfg = TrainFrameConfig(n_world=64, n_screen=64, seed=5)
        got = [train_frame(ps, ps.camera, c, cfg, frame=f) for f in range(3)]
        np.testing.assert_allclose(got, g_train["pen_loss"], rtol=1e-4)

    def test_sharded_grid_gradient_equals_full_batch(self, pbox8, g_train):
        """Fixed-point grid gradients: sum over row shards == full batch, bit for bit."""
        pos = torch.from_numpy(g_train["c1_pos"]).to(DEV)
        tgt = torch.from_numpy(g_train["c1_tgt"].astype(np.float32)).to(DEV)
        full, parts = self._c1(pbox8), self._c1(pbox8)
        full.set_compact(False)
        parts.set_compact(False)
        full.accumulate_grads(pos, tgt)
        b = pos.shape[0]
        for sh in range(4):
            lo, hi = b * sh // 4, b * (sh + 1) // 4
            parts.accumulate_grads(pos, tgt[lo:hi].contiguous(), b_max=b, shard=sh, n_shards=4)
        gc = full.grid_cfg.param_count
        np.testing.assert_array_equal(full.grad_fx[:gc].cpu().numpy(), parts.grad_fx[:gc].cpu().numpy())
        # 4 shards of 8192 rows are 32-row aligned: per-block fixed point makes the
        # MLP gradient shard-exact too
        np.testing.assert_array_equal(full.grad_fx[gc:].cpu().numpy(), parts.grad_fx[gc:].cpu().numpy())


def test_odd_light_count_mixed_emitters():
    """K = 5 (three rect + two point lights): the per-light reservoir paths (K % 4 != 0),
    shading, the training batch and its shadow-ray targets against the oracle."""
    from paper_2506_05930_b200.render import gbuffer_device, shade_batch
    from paper_2506_05930_b200.training import BatchBuffers, gen_batch_device
    d = boxes_scene(8)
    lights = d["lights"][:5]
    for i in (1, 3):
        lt = lights[i]
        c, u, v = (np.array(lt[k], float) for k in ("corner", "edge_u", "edge_v"))
        area = float(np.linalg.norm(np.cross(u, v)))
        lights[i] = {"type": "point", "position": list(c + 0.5 * u + 0.5 * v),
                     "intensity": [area * r for r in lt["radiance"]]}
    d["lights"] = lights
    s = scene_from_dict(d)
    cam = s.camera.resized(48, 32)
    sa = O.SceneArrays(s.triangles_v0, s.triangles_v1, s.triangles_v2, s.tri_material, s.tri_light, s.lt_kind,
                       s.lt_verts, s.lt_normal, s.lt_radiance, s.mat_albedo,
                       np.array([*cam.position, *cam.look_at, *cam.up, cam.fov_deg, cam.width, cam.height], float),
                       lt_area=s.lt_area)
    pos, nrm, alb, _, _ = gbuffer_device(s, cam)
    ctx = PixelCtx(s, pos, nrm, alb)
    c = VisibilityCache(MODE_LIGHTS, 5, grid_cfg(s, 8, 1 << 14), seed=2, hidden_dims=(64, 64))
    c.grid_params = (np.random.default_rng(6).standard_normal(c.grid_params.shape) * 0.5).astype(np.float32)
    vis16 = c.infer(pos.cpu().numpy(), precision=PRECISION_FP16)
    key = R.stream_key(0, 4, "light-select")
    for offset in (0, 2):
        oi, op, ow = O.nls_sample(sa, vis16, ctx.lum_matrix(), key, offset=offset)
        ids, pts, big_w = nls_sample_batch(ctx, c, R.Stream(key=key, offset=offset))
        np.testing.assert_array_equal(ids, oi)
        np.testing.assert_array_equal(pts, op)
        np.testing.assert_array_equal(big_w, ow)
    assert set(np.unique(ids)) >= {1, 3} and (ids >= 0).sum() > 100
    p_h, n_h, a_h = (t.cpu().numpy() for t in (pos, nrm, alb))
    np.testing.assert_array_equal(shade_batch(s, p_h, n_h, a_h, ids, pts, big_w),
                                  O.shade(sa, p_h, n_h, a_h, ids, pts, big_w))
    bufs = BatchBuffers(256, 256, 5, DEV, 1)
    gen_batch_device(s, cam, bufs, 3, 1, 0, 0, 1)
    opos, otgt = O.train_batch(sa, 3, 1, 0, n_world=256, n_screen=256)
    b = int(bufs.n_rows.item())
    np.testing.assert_array_equal(bufs.pos[:b].cpu().numpy(), opos)
    np.testing.assert_array_equal(bufs.tgt[:b].cpu().numpy(), otgt)


@pytest.fixture(scope="module")
def rooms():
    """rooms128 and its 16 k-means light clusters (the reference's clustering stream)."""
    from paper_2506_05930_b200.clusters import kmeans_cluster
    from paper_2506_05930_b200.scenes import rooms_scene
    s = scene_from_dict(rooms_scene(128))
    return s, kmeans_cluster(s.lights, 16, R.stream(0, R.CLUSTERING))


class TestClusters:
    """Clustered NVC on the device (training.py:121-128, sampling.py:302-352)."""

    @pytest.mark.parametrize("walk", [False, True])
    def test_cluster_targets_bit_exact_and_stream_state(self, rooms, g_clusters, walk, monkeypatch):
        """Parallel no-rejection fast path, and the exact sequential walk forced on."""
        if walk:
            monkeypatch.setenv("NVC_CLUSTER_EXACT_WALK", "1")
        s, cs = rooms
        g = R.stream(0, 2, 0, R.TARGETS)
        tgt = compute_visibility_targets(g_clusters["ct_pos"], s, g, clusters=cs)
        np.testing.assert_array_equal(tgt, g_clusters["ct_tgt"])
        # the generator continues exactly where the reference's would (incl. the kept half)
        h = R.stream(0, 2, 0, R.TARGETS)
        b = g_clusters["ct_pos"].shape[0]
        for mem in cs.members:
            h.integers(0, mem.size, size=b)
            h.random((b, 2))
        np.testing.assert_array_equal(g.integers(0, 7, size=9), h.integers(0, 7, size=9))
        np.testing.assert_array_equal(g.random(5), h.random(5))

    def test_targets_continue_a_used_stream(self, rooms, g_scenes):
        """compute_visibility_targets on a Generator that has already drawn -- at an odd
        position and holding a kept 32-bit half -- matches the same numpy calls
        made in the reference's order, and leaves the stream where they do."""
        s, cs = rooms
        sa = O.SceneArrays.from_golden(g_scenes, "rooms128_")
        pos = np.random.default_rng(2).uniform(s.aabb_min, s.aabb_max, (301, 3))
        g, h = R.stream(7, "used"), R.stream(7, "used")
        for x in (g, h):
            x.random(5)
            x.integers(0, 3, size=1)               # leaves a kept half in the bit generator
        tg = compute_visibility_targets(pos, s, g, clusters=cs)
        want = np.empty_like(tg)
        for j, mem in enumerate(cs.members):       # training.py:121-128 with the same generator
            ids = mem[h.integers(0, mem.size, size=pos.shape[0])]
            want[:, j] = sa.visibility(pos, sa.light_points(ids, h.random((pos.shape[0], 2))))
        np.testing.assert_array_equal(tg, want)
        np.testing.assert_array_equal(g.integers(0, 11, size=7), h.integers(0, 11, size=7))
        np.testing.assert_array_equal(g.random(3), h.random(3))
        # light mode from an odd position
        g.random(1)
        h.random(1)
        tl = compute_visibility_targets(pos, s, g)
        wl = np.empty_like(tl)
        for j in range(s.lt_kind.shape[0]):
            wl[:, j] = sa.visibility(pos, sa.light_points(np.full(pos.shape[0], j), h.random((pos.shape[0], 2))))
        np.testing.assert_array_equal(tl, wl)
        np.testing.assert_array_equal(g.random(3), h.random(3))

    def test_rejection_loop_and_kept_half(self, rooms, g_scenes):
        """A 1,431,655,766-member cluster (2^32 mod n = n - 2) rejects a third of its
        32-bit draws, running the multi-window path; a 3-member cluster follows."""
        s, _ = rooms
        from paper_2506_05930_b200.scene import device_scene
        ds = device_scene(s, DEV)
        n_big, b, k = 1431655766, 2001, s.lt_kind.shape[0]
        c_mem = torch.cat([torch.arange(n_big, device=DEV, dtype=torch.int64).remainder_(k).to(torch.int32),
                           torch.tensor([5, 77, 101], dtype=torch.int32, device=DEV)])
        c_off = torch.tensor([0, n_big, n_big + 3], dtype=torch.int32, device=DEV)
        pos_h = np.random.default_rng(1).uniform(s.aabb_min, s.aabb_max, (b, 3))
        pos = torch.from_numpy(pos_h).to(DEV)
        n_rows = torch.tensor([b], dtype=torch.int64, device=DEV)
        tgt = torch.zeros((b + 1, 2), dtype=torch.float32, device=DEV)
        ws = torch.zeros(_lib.load().nvc_cluster_workspace_bytes(b, 2), dtype=torch.uint8, device=DEV)
        key = R.stream_key(4, "reject")
        _lib.call("nvc_cluster_targets", ds.struct, key, 0, -1, pos.data_ptr(), n_rows.data_ptr(), b, 0, 1, 2,
                  c_off.data_ptr(), c_mem.data_ptr(), tgt.data_ptr(), ws.data_ptr(), _lib.stream_ptr())
        del c_mem
        got = tgt[:b].cpu().numpy()
        st = ws.view(torch.int64)[_lib.load().nvc_cluster_state_offset(b, 2) // 8:][:4].cpu().numpy()
        sa = O.SceneArrays.from_golden(g_scenes, "rooms128_")
        pick, used, pend = O.bounded_ints(key, 0, b, n_big)
        assert used > (b + 1) // 2 + 200                         # many rejections
        u = O.uniform_at(key, used + np.arange(2 * b)).reshape(b, 2)
        want0 = sa.visibility(pos_h, sa.light_points(pick % k, u))
        pick2, used2, pend2 = O.bounded_ints(key, used + 2 * b, b, 3, pend)
        u2 = O.uniform_at(key, used + 2 * b + used2 + np.arange(2 * b)).reshape(b, 2)
        want1 = sa.visibility(pos_h, sa.light_points(np.array([5, 77, 101])[pick2], u2))
        np.testing.assert_array_equal(got[:, 0], want0)
        np.testing.assert_array_equal(got[:, 1], want1)
        assert st[0] == used and st[1] == used + 2 * b + used2
        assert st[2] == used + 2 * b + used2 + 2 * b and st[3] == (-1 if pend2 is None else pend2)

    def test_sharded_cluster_targets_equal_whole_batch(self, rooms):
        """Data-parallel shards of a cluster-mode batch: every rank draws the global
        picks and keeps its rows -- concatenated, they equal the unsharded targets."""
        from paper_2506_05930_b200.training import BatchBuffers, gen_batch_device
        s, cs = rooms
        whole = BatchBuffers(1024, 1024, cs.m, DEV, 1)
        gen_batch_device(s, s.camera, whole, 0, 4, 0, 0, 1, clusters=cs)
        b = int(whole.n_rows.item())
        parts = []
        for sh in range(3):
            bufs = BatchBuffers(1024, 1024, cs.m, DEV, 3)
            gen_batch_device(s, s.camera, bufs, 0, 4, 0, sh, 3, clusters=cs)
            lo, hi = b * sh // 3, b * (sh + 1) // 3
            parts.append(bufs.tgt[:hi - lo].cpu().numpy())
        np.testing.assert_array_equal(np.concatenate(parts), whole.tgt[:b].cpu().numpy())

    def test_cluster_train_frame_first_step(self, rooms):
        """A cluster-mode cache trains on cluster targets: first-step loss equals the
        oracle's on the oracle's batch (C-config batch scaled down)."""
        from paper_2506_05930_b200 import make_cache
        from paper_2506_05930_b200.hashgrid import clustered_config
        s, cs = rooms
        cfg = TrainFrameConfig.clustered(n_world=1024, n_screen=1024)
        c = make_cache(s, "clusters", seed=0, clusters=cs.m)
        loss = train_frame(s, s.camera, c, cfg, frame=0, clusters=cs)
        g = clustered_config(aabb_min=s.aabb_min, aabb_max=s.aabb_max)
        oc = O.Cache(O.Grid(levels=g.levels, base_resolution=g.base_resolution, per_level_scale=g.per_level_scale,
                            features_per_level=g.features_per_level, table_size=g.table_size,
                            aabb_min=s.aabb_min, aabb_max=s.aabb_max), cs.m, hidden=c.net_cfg.hidden_dims, seed=0)
        cam = s.camera
        sa = O.SceneArrays(s.triangles_v0, s.triangles_v1, s.triangles_v2, s.tri_material, s.tri_light, s.lt_kind,
                           s.lt_verts, s.lt_normal, s.lt_radiance, s.mat_albedo,
                           np.array([*cam.position, *cam.look_at, *cam.up, cam.fov_deg, cam.width, cam.height], float))
        world = O.world_samples(sa, 1024, O.Stream(0, 0, 0, "world-samples"))
        screen = O.screen_samples(sa, 1024, O.Stream(0, 0, 0, "screen-samples"))
        pos = np.concatenate([world, screen])
        off, flat = cs.packed()
        tgt = O.cluster_targets(sa, pos, np.diff(off), flat, O.stream_key(0, 0, 0, "targets"))
        oloss = oc.train_step(pos, tgt)
        assert abs(loss - oloss) <= 1e-5 * abs(oloss), (loss, oloss)
        with pytest.raises(ValueError):
            train_frame(s, s.camera, c, cfg, frame=1)


class TestClusteredSampling:
    """Two-step clustered light sampling (sampling.py:302-352) on the device."""

    def test_vs_reference_golden(self, rooms, g_clusters):
        from paper_2506_05930_b200 import clustered_sample_batch
        s, cs = rooms
        z = g_clusters
        ctx = PixelCtx(s, z["cs_gb_position"], z["cs_gb_normal"], z["cs_gb_albedo"])
        g = R.stream(0, 3, R.LIGHT_SELECT)
        ids, pts, big_w = clustered_sample_batch(ctx, FixedCache(z["cs_vis"]), cs, g)
        np.testing.assert_array_equal(ids, z["cs_ids"])
        np.testing.assert_array_equal(pts, z["cs_pts"])
        np.testing.assert_allclose(big_w, z["cs_W"], rtol=1e-9, atol=0)   # factors: numba vs FP64 CUDA ~1e-12
        # the stream advanced past step 1 (P*m), step 2 (sum_j n_j |mem_j|) and the points (2P)
        key = R.stream_key(0, 3, R.LIGHT_SELECT)
        c_idx, _, _ = O.wrs_select(np.maximum(z["cs_vis"].astype(np.float64), 0.001), key)
        n_j = np.bincount(c_idx[c_idx >= 0], minlength=cs.m)
        want = ctx.n * cs.m + int(sum(n_j[j] * cs.members[j].size for j in range(cs.m))) + 2 * ctx.n
        assert R.position(g)[1] == want

    @pytest.mark.parametrize("table", ["f32", "f64", "f64_light_major"])
    def test_native_cluster_cache_vs_oracle(self, rooms, g_scenes, table, monkeypatch):
        """Per-(pixel, member) factors computed in the kernel (f32 table context), read
        from the cluster-ordered pixel-major copy of the per-camera f64 factor table
        (default), or read from the light-major table itself: same results."""
        from paper_2506_05930_b200 import clustered_sample_batch, make_cache
        from paper_2506_05930_b200.render import gbuffer_device
        if table == "f64_light_major":
            monkeypatch.setenv("NVC_CLUSTER_LIGHT_MAJOR", "1")
        table = np.float32 if table == "f32" else np.float64
        s, cs = rooms
        pos, nrm, alb, _, _ = gbuffer_device(s, s.camera.resized(80, 45))
        ctx = PixelCtx(s, pos, nrm, alb, table_dtype=table)
        c = make_cache(s, "clusters", seed=1, clusters=cs.m)
        c.grid_params = (np.random.default_rng(3).standard_normal(c.grid_params.shape) * 0.5).astype(np.float32)
        vis = c.infer(pos.cpu().numpy())
        sa = O.SceneArrays.from_golden(g_scenes, "rooms128_")
        off, flat = cs.packed()
        p_h, n_h, a_h = (t.cpu().numpy() for t in (pos, nrm, alb))
        key = R.stream_key(0, 9, R.LIGHT_SELECT)
        for floor in (0.001, 0.0):
            oi, op, ow = O.clustered_sample(sa, vis, sa.factors(p_h, n_h), a_h, np.diff(off), flat, key, floor=floor)
            ids, pts, big_w = clustered_sample_batch(ctx, c, cs, R.Stream(key=key), clamp_floor=floor)
            np.testing.assert_array_equal(ids, oi)
            np.testing.assert_array_equal(pts, op)
            np.testing.assert_allclose(big_w, ow, rtol=1e-9, atol=0)
            assert (ids >= 0).sum() > 1000


def test_snapshot_roundtrip(tmp_path, boxes32):
    c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(boxes32, 8, 1 << 14), hidden_dims=(64, 64))
    c.step = 7
    c.save(tmp_path / "s.vc")
    d = VisibilityCache.load(tmp_path / "s.vc")
    assert d.step == 7 and d.net_cfg.hidden_dims == (64, 64)
    np.testing.assert_array_equal(c.params.cpu().numpy(), d.params.cpu().numpy())
    pos = np.random.default_rng(0).uniform(-1, 1, (300, 3))
    np.testing.assert_array_equal(c.infer(pos), d.infer(pos))


def test_reference_snapshot_interop(tmp_path, g_snap):
    """VCSNAP1 both ways: a snapshot the reference wrote loads here and infers its
    values; our re-save carries byte-identical arrays and every header field the
    reference's loader reads (cache.py:77-117)."""
    import os
    from conftest import read_vcsnap
    ref = os.path.join(os.path.dirname(__file__), "golden", "ref_snapshot.vcsnap")
    c = VisibilityCache.load(ref)
    assert c.step == int(g_snap["snap_step"]) and c.net_cfg.hidden_dims == (32, 32)
    np.testing.assert_allclose(c.infer(g_snap["snap_pos"], precision=PRECISION_FP32), g_snap["snap_infer"],
                               rtol=0, atol=1e-6)
    c.save(tmp_path / "again.vcsnap")
    h0, a0 = read_vcsnap(ref)
    h1, a1 = read_vcsnap(tmp_path / "again.vcsnap")
    for k in ("mode", "output_dim", "step", "grid", "train", "arrays"):
        assert h1[k] == h0[k], k
    for k in a0:
        np.testing.assert_array_equal(a1[k], a0[k])


def test_native_library_is_loaded():
    import ctypes  # noqa: F401
    lib = _lib.load()
    assert lib.nvc_abi_version() == _lib.ABI_VERSION


# ---------------------------------------------------------------------------
# The reference's functional API (hashgrid.py:75-164, mlp.py:110-218,
# training.py:67-94) on the device kernels
# ---------------------------------------------------------------------------
class TestFunctionalApi:
    def _grid(self, scene, levels=8, tsize=1 << 12):
        from paper_2506_05930_b200 import hashgrid as H
        cfg = grid_cfg(scene, levels, tsize)
        og = O.Grid(levels=levels, features_per_level=2, table_size=tsize, aabb_min=scene.aabb_min,
                    aabb_max=scene.aabb_max)
        table = H.init_params(cfg, R.stream(2, "init-params"))
        return H, cfg, og, table

    def test_encode_batch_and_ctx_bit_exact(self, boxes32):
        H, cfg, og, table = self._grid(boxes32)
        pos = R.stream(3, "fn-enc").uniform(boxes32.aabb_min - 0.1, boxes32.aabb_max + 0.1, (3000, 3))
        feats, ctx = H.encode_batch(pos, cfg, table)
        want, wctx = O.encode(og, table, pos)
        np.testing.assert_array_equal(feats, want)
        assert len(ctx) == cfg.levels
        for (i, w), (wi, ww) in zip(ctx, wctx):
            assert i.dtype == np.int64 and i.shape == (3000, 8)
            np.testing.assert_array_equal(i, wi)
            np.testing.assert_array_equal(w, ww)
        np.testing.assert_array_equal(H.encode(pos[5], cfg, table), want[5])
        np.testing.assert_array_equal(H.spatial_hash(np.array([[3, 5, 7]]), 1 << 12),
                                      (3 + 5 * 2654435761 + 7 * 805459861) & 4095)
        with pytest.raises(ValueError):
            H.encode_batch(pos, cfg, table.astype(np.float64))

    @pytest.mark.parametrize("b", [1, 777, 5000])
    def test_grad_from_ctx_bit_exact(self, boxes32, b):
        """np.add.at order (sequential float32 per entry), incl. chunked batches and
        heavy collisions on the coarse dense levels."""
        H, cfg, og, table = self._grid(boxes32)
        pos = R.stream(4, "fn-grad").uniform(boxes32.aabb_min, boxes32.aabb_max, (b, 3))
        up = R.stream(5, "fn-up").normal(0.0, 1.0, (b, cfg.output_dim)).astype(np.float32)
        _, ctx = H.encode_batch(pos, cfg, table)
        got = H.grad_from_ctx(cfg, ctx, up)
        _, wctx = O.encode(og, table, pos)
        np.testing.assert_array_equal(got, O.grid_grad(og, wctx, up))
        np.testing.assert_array_equal(H.encode_backward(pos, cfg, table, up), got)

    def test_mlp_forward_backward_adam(self):
        from paper_2506_05930_b200 import mlp as M
        cfg = M.MLPConfig(input_dim=16, output_dim=8, hidden_dims=(64, 64))
        p = M.he_init(cfg, R.stream(0, "init-params"))
        x = R.stream(6, "fn-x").normal(0.0, 0.5, (513, 16)).astype(np.float32)
        t = (R.stream(7, "fn-t").random((513, 8)) > 0.5).astype(np.float32)
        mask = (R.stream(8, "fn-m").random((513, 8)) > 0.2).astype(np.float32)
        out, cache = M.forward(p, cfg, x)
        wout, zs, acts = O.mlp_forward(p.weights, p.biases, x)
        np.testing.assert_allclose(out, wout, rtol=0, atol=1e-6)        # test_mlp.py:70 tolerance
        assert set(cache) == {"zs", "acts", "out_raw"} and len(cache["zs"]) == 3
        assert M.l2_loss(out, t, mask) == pytest.approx(O.l2_loss(wout, t, mask), rel=1e-5)
        g, d_in = M.backward_l2(p, cfg, cache, t, mask)
        gw, gb, wd = O.mlp_backward(p.weights, zs, acts, t, mask)
        for a, b_ in zip(g.weights + g.biases, gw + gb):
            np.testing.assert_allclose(a, b_, rtol=1e-4, atol=1e-7)
        np.testing.assert_allclose(d_in, wd, rtol=1e-4, atol=1e-7)
        with pytest.raises(ValueError):
            M.forward(p, cfg, np.full((2, 16), np.nan, np.float32))
        with pytest.raises(ValueError):
            M.forward(p, cfg, np.zeros((2, 15), np.float32))
        # Adam: reference op order in float32, bit-exact against the oracle's numpy steps
        params = {k: v.copy() for k, v in p.as_dict().items()}
        st = M.AdamState.for_params(params)
        flat = np.concatenate([v.reshape(-1) for v in params.values()])
        oa = O.Adam(flat.size)
        for step in range(3):
            grads = {k: R.stream(9, step, k).normal(0.0, 1e-2, v.shape).astype(np.float32) for k, v in params.items()}
            M.adam_step(params, grads, st, 0.05)
            oa.step(flat, np.concatenate([grads[k].reshape(-1) for k in params]), 0.05)
        np.testing.assert_array_equal(np.concatenate([v.reshape(-1) for v in params.values()]), flat)
        assert st.t == 3

    def test_gen_screen_hits_matches_reference(self, boxes8, g_scenes):
        from paper_2506_05930_b200.training import gen_screen_hits
        g = R.stream(11, "hits")
        pos, nrm, alb, is_light = gen_screen_hits(boxes8, boxes8.camera, 400, g)
        sa = O.SceneArrays.from_golden(g_scenes, "boxes8_")
        st = O.Stream(key=R.stream_key(11, "hits"))
        w, h = boxes8.camera.width, boxes8.camera.height
        want = {"position": [], "normal": [], "albedo": [], "light": []}
        left = 400
        for _ in range(9):
            if left == 0:
                break
            sx = st.random(left) * w
            sy = st.random(left) * h
            tr = sa.trace(*sa.camera_rays(sx, sy))
            for k in ("position", "normal", "albedo"):
                want[k].append(tr[k][tr["hit"]])
            want["light"].append(tr["light_id"][tr["hit"]] >= 0)
            left -= int(tr["hit"].sum())
        np.testing.assert_array_equal(pos, np.concatenate(want["position"]))
        np.testing.assert_array_equal(nrm, np.concatenate(want["normal"]))
        np.testing.assert_array_equal(alb, np.concatenate(want["albedo"]))
        np.testing.assert_array_equal(is_light, np.concatenate(want["light"]))
        np.testing.assert_array_equal(g.random(2), O.uniform_at(st.key, st.offset + np.arange(2)))
        np.testing.assert_array_equal(gen_screen_samples(boxes8, boxes8.camera, 400, R.stream(11, "hits")), pos)
