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
