"""Pin the CPU oracle against the golden vectors the REFERENCE produced
(tests/golden/make_golden.py).  CPU only; this is what makes the oracle
trustworthy as the checker for the CUDA path."""

import hashlib

import numpy as np
import pytest

from oracle import vc_oracle as O

DEFAULT_SCALE = (512.0 / 16.0) ** (1.0 / 9.0)


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


PARTS = [(0,), (7,), (0, "init-params"), (0, 3, "light-select"), (5, 2, 1, "targets"),
         ("primary",), (123456789012345, -3, "x"), (2**64 - 1, 2**63)]


class TestRng:
    def test_stream_keys(self, g_rng):
        keys = [O.stream_key(*p) for p in PARTS]
        assert keys == [int(k) for k in g_rng["rng_keys"]]

    def test_first_draws_bit_exact(self, g_rng):
        for p, want in zip(PARTS, g_rng["rng_first"]):
            got = O.Stream(*p).random(41)
            np.testing.assert_array_equal(got, want)

    def test_raw_words(self, g_rng):
        got = O.raw_at(O.stream_key(0, 3, "light-select"), np.arange(16))
        np.testing.assert_array_equal(got, g_rng["rng_raw"])

    def test_random_access(self, g_rng):
        key = O.stream_key(0, 3, "light-select")
        np.testing.assert_array_equal(O.uniform_at(key, np.arange(1001, 1011)), g_rng["rng_at1001"])

    def test_uniform_broadcast(self, g_rng):
        st = O.Stream(9, 1, 0, "world-samples")
        got = st.uniform(np.array([-3.0, 0.0, -2.2]), np.array([3.0, 1.5, 3.0]), (5, 3))
        np.testing.assert_array_equal(got, g_rng["rng_uniform"])


def scene(g_scenes, name):
    return O.SceneArrays.from_golden(g_scenes, name + "_")


class TestScene:
    @pytest.mark.parametrize("name", ["boxes8", "boxes32", "rooms128", "pbox8"])
    def test_bvh_matches_reference(self, g_scenes, name):
        s = scene(g_scenes, name)
        np.testing.assert_array_equal(s.bvh.perm, g_scenes[name + "_bvh_perm"])
        np.testing.assert_array_equal(s.bvh.node_min, g_scenes[name + "_bvh_node_min"])
        np.testing.assert_array_equal(s.bvh.left, g_scenes[name + "_bvh_node_left"])
        np.testing.assert_array_equal(s.aabb_min, g_scenes[name + "_aabb_min"])
        np.testing.assert_array_equal(s.aabb_max, g_scenes[name + "_aabb_max"])


def grid_for(g_hash, tag, levels, tsize, g_scenes):
    s = scene(g_scenes, "boxes32")
    return O.Grid(levels=levels, features_per_level=2, table_size=tsize,
                  aabb_min=s.aabb_min, aabb_max=s.aabb_max)


@pytest.mark.parametrize("tag,levels,tsize,seed", [("hc1", 8, 1 << 14, 0), ("hc2", 16, 1 << 19, 1)])
class TestHashGrid:
    def test_resolutions(self, g_hash, g_scenes, tag, levels, tsize, seed):
        g = grid_for(g_hash, tag, levels, tsize, g_scenes)
        assert [g.res(l) for l in range(levels)] == list(g_hash[tag + "_res"])
        assert [g.dense(l) for l in range(levels)] == list(g_hash[tag + "_dense"])

    def test_indices_and_weights_bit_exact(self, g_hash, g_scenes, tag, levels, tsize, seed):
        g = grid_for(g_hash, tag, levels, tsize, g_scenes)
        q = O.normalize(g, g_hash[tag + "_pos"])
        for l in range(levels):
            idx, w = O.level_lookup(g, l, q)
            np.testing.assert_array_equal(idx, g_hash[tag + "_idx"][:, l])
            np.testing.assert_array_equal(w, g_hash[tag + "_w"][:, l])

    def test_features_bit_exact(self, g_hash, g_scenes, tag, levels, tsize, seed):
        g = grid_for(g_hash, tag, levels, tsize, g_scenes)
        c = O.Cache(g, 4, seed=seed)
        assert sha(c.table) == str(g_hash[tag + "_table_sha"])
        feats, ctx = O.encode(g, c.table, g_hash[tag + "_pos"])
        np.testing.assert_array_equal(feats, g_hash[tag + "_feats"])

    def test_grid_grad_bit_exact(self, g_hash, g_scenes, tag, levels, tsize, seed):
        g = grid_for(g_hash, tag, levels, tsize, g_scenes)
        c = O.Cache(g, 4, seed=seed)
        _, ctx = O.encode(g, c.table, g_hash[tag + "_pos"])
        grad = O.grid_grad(g, ctx, g_hash[tag + "_up"]).reshape(-1)
        nz = np.flatnonzero(grad)
        np.testing.assert_array_equal(nz, g_hash[tag + "_grad_nz"])
        np.testing.assert_array_equal(grad[nz], g_hash[tag + "_grad_val"])


class TestMlp:
    def _params(self, g_mlp):
        ws = [g_mlp[f"mlp_w{i}"] for i in range(3)]
        bs = [g_mlp[f"mlp_b{i}"] for i in range(3)]
        return ws, bs

    def test_he_init_stream(self, g_mlp):
        gen = np.random.Generator(np.random.Philox(key=O.stream_key(3, "golden-mlp")))
        ws, _ = O.he_weights([16, 64, 64, 8], gen)
        for i in range(3):
            np.testing.assert_array_equal(ws[i], g_mlp[f"mlp_w{i}"])

    def test_forward_backward(self, g_mlp):
        ws, bs = self._params(g_mlp)
        out, zs, acts = O.mlp_forward(ws, bs, g_mlp["mlp_x"])
        np.testing.assert_allclose(out, g_mlp["mlp_y"], rtol=0, atol=1e-6)
        assert O.l2_loss(out, g_mlp["mlp_t"]) == pytest.approx(float(g_mlp["mlp_loss"]), rel=1e-6)
        gw, gb, dx = O.mlp_backward(ws, zs, acts, g_mlp["mlp_t"])
        for i in range(3):
            np.testing.assert_allclose(gw[i], g_mlp[f"mlp_gw{i}"], rtol=1e-4, atol=1e-9)
            np.testing.assert_allclose(gb[i], g_mlp[f"mlp_gb{i}"], rtol=1e-4, atol=1e-9)
        np.testing.assert_allclose(dx, g_mlp["mlp_dx"], rtol=1e-4, atol=1e-10)

    def test_adam_trajectory_bit_exact(self, g_mlp):
        p = g_mlp["adam_p0"].copy()
        st = O.Adam(p.size)
        for i, lr in enumerate(g_mlp["adam_lr"]):
            st.step(p, g_mlp["adam_g"][i], float(lr))
            np.testing.assert_array_equal(p, g_mlp["adam_traj"][i])
        np.testing.assert_array_equal(st.m, g_mlp["adam_m"])
        np.testing.assert_array_equal(st.v, g_mlp["adam_v"])

    def test_lr_schedule(self):
        assert O.lr_at(0) == 0.05 and O.lr_at(200) == pytest.approx(0.001)
        assert O.lr_at(10_000) == O.lr_at(200)


class TestGeometry:
    def test_gbuffer_bit_exact(self, g_scenes, g_samp):
        s = scene(g_scenes, "boxes32")
        gb = s.gbuffer(40, 24)
        np.testing.assert_array_equal(gb["hit"], g_samp["gb_hit"])
        np.testing.assert_array_equal(gb["position"], g_samp["gb_position"])
        np.testing.assert_array_equal(gb["normal"], g_samp["gb_normal"])
        np.testing.assert_array_equal(gb["albedo"], g_samp["gb_albedo"])
        np.testing.assert_array_equal(gb["light_id"], g_samp["gb_light_id"])

    def test_point_scene_gbuffer_and_factors(self, g_scenes, g_samp):
        s = scene(g_scenes, "pbox8")
        gb = s.gbuffer()
        np.testing.assert_array_equal(gb["position"], g_samp["pgb_position"])
        f = s.factors(gb["position"], gb["normal"])
        np.testing.assert_allclose(f, g_samp["pgb_factor"], rtol=1e-12, atol=0)

    def test_rect_factors(self, g_scenes, g_samp):
        s = scene(g_scenes, "boxes32")
        f = s.factors(g_samp["gb_position"], g_samp["gb_normal"])
        np.testing.assert_allclose(f, g_samp["nls_factor"], rtol=1e-10, atol=1e-300)
        lum = s.lum(g_samp["nls_factor"], g_samp["gb_albedo"])
        np.testing.assert_array_equal(lum, g_samp["nls_lum"])

    def test_visibility_segments(self, g_scenes, g_train):
        s = scene(g_scenes, "boxes32")
        np.testing.assert_array_equal(s.visibility(g_train["vis_x"], g_train["vis_y"]),
                                      g_train["vis_b32"])


class TestTrainingData:
    def test_screen_samples_bit_exact(self, g_scenes, g_train):
        s = scene(g_scenes, "boxes8")
        got = O.screen_samples(s, 256, O.Stream(6))
        np.testing.assert_array_equal(got, g_train["screen_boxes8_256"])

    def test_c1_batch_and_targets_bit_exact(self, g_scenes, g_train):
        s = scene(g_scenes, "pbox8")
        pos, tgt = O.train_batch(s, 0, 0)
        np.testing.assert_array_equal(pos, g_train["c1_pos"])
        np.testing.assert_array_equal(tgt.astype(np.uint8), g_train["c1_tgt"])

    def test_boxes32_targets_bit_exact(self, g_scenes, g_train):
        s = scene(g_scenes, "boxes32")
        pos, tgt = O.train_batch(s, 0, 3, n_world=2048, n_screen=2048)
        np.testing.assert_array_equal(pos, g_train["b32_pos"])
        np.testing.assert_array_equal(tgt.astype(np.uint8), g_train["b32_tgt"])


class TestSampling:
    def test_wrs_bit_exact(self, g_samp):
        key = O.stream_key(0, 4, "light-select")
        w = g_samp["wrs_w"]
        idx, wsel, wsum = O.wrs_select(w, key)
        np.testing.assert_array_equal(idx, g_samp["wrs_idx"])
        np.testing.assert_array_equal(wsel, g_samp["wrs_wsel"])
        np.testing.assert_array_equal(wsum, g_samp["wrs_wsum"])
        idx2, _, _ = O.wrs_select(w[:17], key, offset=w.size)
        np.testing.assert_array_equal(idx2, g_samp["wrs_idx2"])

    def test_nls_bit_exact(self, g_scenes, g_samp):
        s = scene(g_scenes, "boxes32")
        key = O.stream_key(0, 7, "light-select")
        ids, pts, big_w = O.nls_sample(s, g_samp["nls_vis"], g_samp["nls_lum"], key)
        np.testing.assert_array_equal(ids, g_samp["nls_ids"])
        np.testing.assert_array_equal(pts, g_samp["nls_pts"])
        np.testing.assert_array_equal(big_w, g_samp["nls_W"])
        ids, _, big_w = O.nls_sample(s, g_samp["nls_vis"], g_samp["nls_lum"], key, floor=0.0)
        np.testing.assert_array_equal(ids, g_samp["nls_ids_biased"])
        np.testing.assert_array_equal(big_w, g_samp["nls_W_biased"])

    def test_nls_sharded_matches_whole(self, g_scenes, g_samp):
        s = scene(g_scenes, "boxes32")
        key = O.stream_key(0, 7, "light-select")
        p = g_samp["nls_vis"].shape[0]
        cuts = [0, 301, 517, p]
        parts = [O.nls_sample(s, g_samp["nls_vis"][a:b], g_samp["nls_lum"][a:b], key,
                              p_total=p, p_first=a) for a, b in zip(cuts[:-1], cuts[1:])]
        np.testing.assert_array_equal(np.concatenate([q[0] for q in parts]), g_samp["nls_ids"])
        np.testing.assert_array_equal(np.concatenate([q[1] for q in parts]), g_samp["nls_pts"])

    def test_neural_di(self, g_scenes, g_samp):
        s = scene(g_scenes, "boxes32")
        rgb = O.neural_di(s, g_samp["nls_vis"], g_samp["nls_factor"], g_samp["gb_albedo"])
        np.testing.assert_allclose(rgb, g_samp["ndi_rgb"], rtol=1e-12, atol=1e-300)


class TestShade:
    """Shading pass 5 (render.py:220-246) against the reference's shade_batch."""

    def test_boxes32_random_samples(self, g_scenes, g_shade):
        s = scene(g_scenes, "boxes32")
        z = g_shade
        rgb = O.shade(s, z["b32_position"], z["b32_normal"], z["b32_albedo"], z["b32_ids"], z["b32_pts"], z["b32_W"])
        np.testing.assert_array_equal(rgb, z["b32_rgb"])
        assert (rgb != 0).any(axis=1).sum() > 100

    def test_point_lights(self, g_scenes, g_samp, g_shade):
        s = scene(g_scenes, "pbox8")
        z = g_shade
        rgb = O.shade(s, g_samp["pgb_position"], g_samp["pgb_normal"], g_samp["pgb_albedo"], z["p8_ids"],
                      z["p8_pts"], z["p8_W"])
        np.testing.assert_array_equal(rgb, z["p8_rgb"])

    def test_nls_samples(self, g_scenes, g_samp, g_shade):
        s = scene(g_scenes, "boxes32")
        rgb = O.shade(s, g_samp["gb_position"], g_samp["gb_normal"], g_samp["gb_albedo"], g_samp["nls_ids"],
                      g_samp["nls_pts"], g_samp["nls_W"])
        np.testing.assert_array_equal(rgb, g_shade["nls_rgb"])


class TestClusters:
    """Clustered NVC (training.py:121-128, sampling.py:302-352) against the reference."""

    def test_bounded_integers_match_numpy(self):
        key = O.stream_key(3, "x")
        for n, cnt, start in ((37, 1001, 0), (2, 7, 5), (1, 10, 3), (1000003, 999, 11)):
            want = np.random.Generator(np.random.Philox(key=key))
            want.random(start) if start else None
            vals, used, pend = O.bounded_ints(key, start, cnt, n)
            np.testing.assert_array_equal(vals, want.integers(0, n, size=cnt))
            np.testing.assert_array_equal(O.uniform_at(key, np.arange(start + used, start + used + 2)), want.random(2))
            more, _, _ = O.bounded_ints(key, start + used + 2, 5, n, pend)   # the kept half carries over
            np.testing.assert_array_equal(more, want.integers(0, n, size=5))

    def test_cluster_targets_bit_exact(self, g_scenes, g_clusters):
        s = scene(g_scenes, "rooms128")
        tgt = O.cluster_targets(s, g_clusters["ct_pos"], g_clusters["km_r128k16_sizes"],
                                g_clusters["km_r128k16_members"], O.stream_key(0, 2, 0, "targets"))
        np.testing.assert_array_equal(tgt, g_clusters["ct_tgt"])
        assert 0.05 < tgt.mean() < 0.95

    def test_clustered_sample(self, g_scenes, g_clusters):
        """ids and points exact; W to 1e-9 (the unshadowed factors restate numba's
        acos/sqrt chain to ~1e-12)."""
        z = g_clusters
        s = scene(g_scenes, "rooms128")
        f = s.factors(z["cs_gb_position"], z["cs_gb_normal"])
        ids, pts, big_w = O.clustered_sample(s, z["cs_vis"], f, z["cs_gb_albedo"], z["km_r128k16_sizes"],
                                             z["km_r128k16_members"], O.stream_key(0, 3, "light-select"))
        np.testing.assert_array_equal(ids, z["cs_ids"])
        np.testing.assert_array_equal(pts, z["cs_pts"])
        np.testing.assert_allclose(big_w, z["cs_W"], rtol=1e-9, atol=0)
        assert (ids >= 0).sum() > 1000


class TestSnapshot:
    def test_reference_snapshot_reads_and_infers(self, g_snap):
        """The reference's VCSNAP1 file, parsed by the restated reader and evaluated by
        the oracle, reproduces the reference cache's infer() (cache.py:54-58, 99-117)."""
        import os
        from conftest import read_vcsnap
        header, arrays = read_vcsnap(os.path.join(os.path.dirname(__file__), "golden", "ref_snapshot.vcsnap"))
        assert header["mode"] == "lights" and header["step"] == int(g_snap["snap_step"])
        gc = header["grid"]
        g = O.Grid(levels=gc["levels"], base_resolution=gc["base_resolution"],
                   per_level_scale=gc["per_level_scale"], features_per_level=gc["features_per_level"],
                   table_size=gc["table_size"], aabb_min=gc["aabb_min"], aabb_max=gc["aabb_max"])
        n = sum(1 for k in arrays if k.startswith("w"))
        feats, _ = O.encode(g, arrays["grid"], g_snap["snap_pos"])
        out, _, _ = O.mlp_forward([arrays[f"w{i}"] for i in range(n)], [arrays[f"b{i}"] for i in range(n)], feats)
        np.testing.assert_allclose(out, g_snap["snap_infer"], rtol=0, atol=1e-6)


class TestTrainingCurve:
    def test_first_step_matches_reference(self, g_scenes, g_train):
        s = scene(g_scenes, "pbox8")
        g = O.Grid(levels=8, features_per_level=2, table_size=1 << 14,
                   aabb_min=s.aabb_min, aabb_max=s.aabb_max)
        c = O.Cache(g, 8, hidden=(64, 64))
        loss = c.train_step(g_train["c1_pos"], g_train["c1_tgt"].astype(np.float32))
        assert loss == pytest.approx(float(g_train["c1_step0_loss"]), rel=1e-6)
        np.testing.assert_allclose(c.ws[0], g_train["c1_step0_w0"], atol=2e-6)

    def test_loss_curve_within_band(self, g_scenes, g_train):
        s = scene(g_scenes, "pbox8")
        g = O.Grid(levels=8, features_per_level=2, table_size=1 << 14,
                   aabb_min=s.aabb_min, aabb_max=s.aabb_max)
        c = O.Cache(g, 8, hidden=(64, 64))
        want = g_train["c1_loss_f32"][:4]
        got = []
        for f in range(len(want)):
            pos, tgt = O.train_batch(s, 0, f)
            got.append(c.train_step(pos, tgt))
        np.testing.assert_allclose(got, want, rtol=2e-3)
