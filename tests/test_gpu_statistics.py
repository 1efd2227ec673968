"""GPU statistical checks mirroring the reference's sampling tests
(viscache tests/test_sampling.py): selection frequencies, the two-step
clustered pmf, and unbiasedness of the clustered estimator through the GPU
shading pass.  These test distributions, not bits -- the bit-level parity of
the same kernels is in test_gpu_parity.py."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
stats = pytest.importorskip("scipy.stats")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import vc_oracle as O  # noqa: E402
from paper_2506_05930_b200 import (PixelCtx, scene_from_dict, wrs_select_batch,  # noqa: E402
                                   clustered_sample_batch, nls_sample_batch, shade_batch)
from paper_2506_05930_b200 import rng as R  # noqa: E402
from paper_2506_05930_b200.clusters import ClusterSet, kmeans_cluster  # noqa: E402
from paper_2506_05930_b200.scenes import boxes_scene, quad  # noqa: E402

LUMA = np.array([0.2126, 0.7152, 0.0722])
FLOOR = quad((-4, 0, -4), (4, 0, -4), (4, 0, 4), (-4, 0, 4))


def down_light(cx, cz, y, size, radiance=(10.0, 10.0, 10.0)):
    h = size / 2.0
    return {"type": "rect", "corner": [cx - h, y, cz - h], "edge_u": [size, 0, 0], "edge_v": [0, 0, size],
            "radiance": list(radiance)}


def make_scene(lights, meshes):
    return scene_from_dict({"camera": {"position": [0, 1.5, 3], "look_at": [0, 0, 0], "up": [0, 1, 0],
                                       "fov_deg": 50.0, "width": 64, "height": 48},
                            "materials": [{"albedo": [0.7, 0.7, 0.7]}], "meshes": meshes, "lights": lights})


@pytest.fixture(scope="module")
def two_cluster_scene():
    plate = quad((-1.4, 1, -0.6), (-0.2, 1, -0.6), (-0.2, 1, 0.6), (-1.4, 1, 0.6))
    lights = [down_light(-2.2 + 0.5 * i, 0.0, 2.0, 0.3, (9.0, 8.0, 7.0)) for i in range(3)]
    lights += [down_light(1.7 + 0.5 * i, 0.0, 2.0, 0.3, (6.0, 8.0, 10.0)) for i in range(3)]
    return make_scene(lights, [{"material": 0, "triangles": FLOOR}, {"material": 0, "triangles": plate}])


class FixedCache:
    def __init__(self, row, mode="lights"):
        self.row = np.asarray(row, np.float32)
        self.mode, self.output_dim = mode, len(self.row)

    def infer(self, positions):
        return np.tile(self.row, (np.atleast_2d(positions).shape[0], 1))


def tiled_ctx(scene, pos, n, nrm=(0.0, 1.0, 0.0)):
    alb = np.array([0.7, 0.7, 0.7])
    return PixelCtx(scene, np.tile(pos, (n, 1)), np.tile(nrm, (n, 1)), np.tile(alb, (n, 1)), table_dtype=np.float64)


def two_clusters(scene):
    cs = kmeans_cluster(scene.lights, 2, R.stream(61))
    if cs.centroids[0][0] > 0:                          # cluster 0 = the lights at negative x
        cs = ClusterSet(centroids=cs.centroids[::-1].copy(), members=list(reversed(cs.members)))
    return cs


def test_wrs_chi_square_32_lights():
    rng = R.stream(46)
    for _ in range(3):
        w = rng.random(32) + 0.05
        idx, _, _ = wrs_select_batch(np.tile(w, (200_000, 1)), rng)
        chi = stats.chisquare(np.bincount(idx, minlength=32), w / w.sum() * 200_000)
        assert chi.pvalue > 0.001


def test_nls_equal_predictions_follow_unshadowed_distribution():
    s = scene_from_dict(boxes_scene(8))
    n = 200_000
    ctx = tiled_ctx(s, (0.4, 0.0, 0.1), n)
    lum = ctx.lum_matrix()[0]
    ids, _, _ = nls_sample_batch(ctx, FixedCache([0.5] * 8), R.stream(50))
    chi = stats.chisquare(np.bincount(ids, minlength=8), lum / lum.sum() * n)
    assert chi.pvalue > 0.001


def test_one_cluster_one_light_has_unit_weight():
    s = make_scene([down_light(0.0, 0.0, 2.0, 1.0)], [{"material": 0, "triangles": FLOOR}])
    cs = ClusterSet(centroids=np.zeros((1, 3)), members=[np.array([0])])
    ids, pts, w = clustered_sample_batch(tiled_ctx(s, (0.0, 0.0, 0.0), 1), FixedCache([0.6], "clusters"), cs,
                                         R.stream(62))
    assert ids[0] == 0 and w[0] == pytest.approx(1.0) and pts[0, 1] == pytest.approx(2.0)


def test_clustered_selection_pmf_matches_composition(two_cluster_scene):
    s, cs = two_cluster_scene, two_clusters(two_cluster_scene)
    n = 1_000_000
    ctx = tiled_ctx(s, (0.5, 0.0, 0.3), n)
    lum = ctx.lum_matrix()[0]
    cw = np.maximum(np.array([0.9, 0.2]), 0.001)
    pmf = np.zeros(6)
    for j, mem in enumerate(cs.members):
        pmf[mem] = (cw[j] / cw.sum()) * lum[mem] / lum[mem].sum()
    ids, _, _ = clustered_sample_batch(ctx, FixedCache([0.9, 0.2], "clusters"), cs, R.stream(63))
    tv = 0.5 * np.abs(np.bincount(ids, minlength=6) / n - pmf).sum()
    assert tv < 0.005


def test_clustered_estimator_unbiased_through_gpu_shading(two_cluster_scene):
    """Two-step selection + one-shadow-ray shading (both on the GPU) vs the
    exhaustive shadowed sum with many area samples per light (CPU oracle)."""
    s, cs = two_cluster_scene, two_clusters(two_cluster_scene)
    probe, nrm = np.array([-0.8, 0.0, 0.0]), np.array([0.0, 1.0, 0.0])
    n = 2_000_000
    ctx = tiled_ctx(s, probe, n)
    ids, pts, w = clustered_sample_batch(ctx, FixedCache([0.35, 0.75], "clusters"), cs, R.stream(64))
    est = shade_batch(s, ctx.positions, np.tile(nrm, (n, 1)), np.tile([0.7, 0.7, 0.7], (n, 1)), ids, pts, w) @ LUMA
    sa = O.SceneArrays(s.triangles_v0, s.triangles_v1, s.triangles_v2, s.tri_material, s.tri_light, s.lt_kind,
                       s.lt_verts, s.lt_normal, s.lt_radiance, s.mat_albedo, np.zeros(12), lt_area=s.lt_area)
    m = 4000
    u = np.random.default_rng(5).random((m, 2))
    total = 0.0
    for k in range(6):
        y = sa.light_points(np.full(m, k), u)
        vis = sa.visibility(np.tile(probe, (m, 1)), y)
        d = y - probe
        d2 = (d * d).sum(axis=1)
        wd = d / np.sqrt(d2)[:, None]
        g = np.maximum(0.0, wd @ nrm) * np.maximum(0.0, -(wd @ s.lt_normal[k])) / d2
        total += float((0.7 / np.pi * s.lt_radiance[k] @ LUMA) * np.mean(g * vis) * s.lt_area[k])
    se = est.std() / np.sqrt(n)
    assert abs(est.mean() - total) < 3 * se + 0.005 * total


def test_cluster_weights_ignore_radiance(two_cluster_scene):
    s, cs = two_cluster_scene, two_clusters(two_cluster_scene)
    n = 50_000
    ids, _, _ = clustered_sample_batch(tiled_ctx(s, (0.0, 0.0, 1.0), n), FixedCache([0.5, 0.5], "clusters"), cs,
                                       R.stream(65))
    assert np.isin(ids, cs.members[0]).mean() == pytest.approx(0.5, abs=0.01)


# ---------------------------------------------------------------------------
# behaviour of training targets, training and shading (reference
# tests/test_training.py, test_render.py, restated on the GPU path)
# ---------------------------------------------------------------------------
def penumbra_scene():
    plate = quad((-0.5, 1, -0.5), (0.5, 1, -0.5), (0.5, 1, 0.5), (-0.5, 1, 0.5))
    return scene_from_dict({"camera": {"position": [0, 1.6, 3.2], "look_at": [0, 0, 0], "up": [0, 1, 0],
                                       "fov_deg": 55.0, "width": 96, "height": 54},
                            "materials": [{"albedo": [0.7, 0.7, 0.7]}, {"albedo": [0.5, 0.3, 0.3]}],
                            "meshes": [{"material": 0, "triangles": FLOOR}, {"material": 1, "triangles": plate}],
                            "lights": [down_light(0.0, 0.0, 2.0, 0.8)]})


def single_light_scene():
    return make_scene([down_light(0.0, 0.0, 2.0, 1.0)], [{"material": 0, "triangles": FLOOR}])


def test_targets_unoccluded_occluded_binary(two_cluster_scene):
    from paper_2506_05930_b200.training import compute_visibility_targets, gen_world_samples
    rng = R.stream(8)
    pts = np.column_stack([rng.uniform(-3, 3, 200), np.zeros(200), rng.uniform(-3, 3, 200)])
    np.testing.assert_array_equal(compute_visibility_targets(pts, single_light_scene(), rng), 1.0)
    under = np.zeros((200, 3))                       # under the plate: umbra
    np.testing.assert_array_equal(compute_visibility_targets(under, penumbra_scene(), R.stream(9)), 0.0)
    s8 = scene_from_dict(boxes_scene(8))
    t = compute_visibility_targets(gen_world_samples(s8, 300, R.stream(10)), s8, R.stream(11))
    assert set(np.unique(t)) <= {0.0, 1.0} and 0.0 < t.mean() < 1.0
    cs = kmeans_cluster(two_cluster_scene.lights, 2, R.stream(13))
    tc = compute_visibility_targets(gen_world_samples(two_cluster_scene, 64, R.stream(14)), two_cluster_scene,
                                    R.stream(15), clusters=cs)
    assert tc.shape == (64, 2) and set(np.unique(tc)) <= {0.0, 1.0}


def test_loss_decreases_frame_to_frame():
    from paper_2506_05930_b200 import TrainFrameConfig, make_cache, train_frame
    s8 = scene_from_dict(boxes_scene(8))
    wins = 0
    for seed in range(20):
        c = make_cache(s8, "lights", seed=seed)
        cfg = TrainFrameConfig(n_world=256, n_screen=256, seed=seed)
        l0 = train_frame(s8, s8.camera, c, cfg, frame=0)
        wins += train_frame(s8, s8.camera, c, cfg, frame=1) <= l0
    assert wins >= 18


def test_converged_prediction_tracks_visibility():
    """512 online frames on the penumbra scene: the umbra predicts ~0, open floor ~1."""
    from paper_2506_05930_b200 import TrainFrameConfig, make_cache, train_frame
    s = penumbra_scene()
    c = make_cache(s, "lights", seed=7)
    cfg = TrainFrameConfig(n_world=512, n_screen=512, seed=7)
    for f in range(512):
        train_frame(s, s.camera, c, cfg, frame=f)
    pred = c.infer(np.array([[0.0, 0.0, 0.0], [3.0, 0.0, 3.0], [-3.0, 0.0, 2.5]]))[:, 0]
    assert pred[0] < 0.15 and pred[1] > 0.85 and pred[2] > 0.85


def test_shading_closed_forms():
    from paper_2506_05930_b200 import ShadingPoint, shade_pixel
    # occluded sample is black
    sp = ShadingPoint(np.zeros(3), np.array([0.0, 1.0, 0.0]), np.array([0.7, 0.7, 0.7]))
    np.testing.assert_array_equal(shade_pixel(sp, (0, np.array([0.0, 2.0, 0.0]), 1.0), penumbra_scene()), 0.0)
    # point light: albedo/pi * I * cos / d^2
    s = make_scene([{"type": "point", "position": [0.0, 2.0, 1.0], "intensity": [5.0, 4.0, 3.0]}],
                   [{"material": 0, "triangles": FLOOR}])
    rgb = shade_pixel(sp, (0, np.array([0.0, 2.0, 1.0]), 1.0), s)
    want = sp.albedo / np.pi * np.array([5.0, 4.0, 3.0]) * (2.0 / np.sqrt(5.0)) / 5.0
    np.testing.assert_allclose(rgb, want, rtol=1e-12)


def test_unoccluded_single_light_estimate_matches_unshadowed_integral():
    """One-light area sampling through shade_batch converges to the analytic
    unshadowed radiance (the factor's closed-form polygon integral)."""
    s = single_light_scene()
    n = 400_000
    ctx = tiled_ctx(s, (0.5, 0.0, 0.5), n)
    u = np.random.default_rng(3).random((n, 2))
    sa = O.SceneArrays(s.triangles_v0, s.triangles_v1, s.triangles_v2, s.tri_material, s.tri_light, s.lt_kind,
                       s.lt_verts, s.lt_normal, s.lt_radiance, s.mat_albedo, np.zeros(12), lt_area=s.lt_area)
    pts = sa.light_points(np.zeros(n, np.int64), u)
    est = shade_batch(s, ctx.positions, np.tile([0.0, 1.0, 0.0], (n, 1)), np.tile([0.7, 0.7, 0.7], (n, 1)),
                      np.zeros(n, np.int64), pts, np.ones(n)) @ LUMA
    want = ctx.lum_matrix()[0, 0]                       # factor * albedo.(LUMA*L)/pi
    se = est.std() / np.sqrt(n)
    assert abs(est.mean() - want) < 4 * se + 1e-3 * want
