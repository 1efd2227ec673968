"""Scalar API wrappers (reference sampling.py:88-101, 141-176, 208-222) against
the reference's own outputs (tests/golden/scalar.npz, make_golden.py
gen_scalar): wrs_select, nls_sample, neural_di_shade, unshadowed_weight,
unshadowed_rgb_one and PixelCtx.phat_ids on 48 boxes8 (rect lights) and 16
point-light shading points.  Integer / selection results bit-exact; FP64
values within 1e-9 relative (the device factor kernel restates numba's acos
chain to ~1e-12)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_05930_b200 import (MODE_LIGHTS, PixelCtx, ShadingPoint, neural_di_shade, nls_sample,  # noqa: E402
                                   scene_from_dict, wrs_select)
from paper_2506_05930_b200 import rng as R  # noqa: E402
from paper_2506_05930_b200.sampling import unshadowed_rgb_one, unshadowed_weight  # noqa: E402
from paper_2506_05930_b200.scenes import boxes_point_scene, boxes_scene  # noqa: E402

from conftest import golden  # noqa: E402

RTOL = 1e-9


class WaveCache:
    """make_golden.WaveCache: visibility = 0.5 + 0.4 sin(a . pos + j)."""
    mode = MODE_LIGHTS

    def __init__(self, k):
        self.output_dim = k

    def infer(self, positions):
        pos = np.atleast_2d(np.asarray(positions, np.float64))
        ph = pos @ np.array([1.3, 2.1, 0.7])
        return (0.5 + 0.4 * np.sin(ph[:, None] + np.arange(self.output_dim))).astype(np.float32)


@pytest.fixture(scope="module")
def g_scalar():
    return golden("scalar")


SCENES = {"b8": lambda: scene_from_dict(boxes_scene(8)), "p8": lambda: scene_from_dict(boxes_point_scene(8))}


@pytest.mark.parametrize("tag", ["b8", "p8"])
def test_scalar_wrappers_vs_reference(g_scalar, tag):
    sc = SCENES[tag]()
    pos, nrm, alb = (g_scalar[f"sc_{tag}_{k}"] for k in ("pos", "nrm", "alb"))
    k = sc.n_lights
    cache = WaveCache(k)
    wts = g_scalar[f"sc_{tag}_wrs_w"]
    for i in range(pos.shape[0]):
        sp = ShadingPoint(position=pos[i], normal=nrm[i], albedo=alb[i])
        r = wrs_select(wts[i], R.stream(0, i, "wrs-scalar"))
        np.testing.assert_array_equal([r.y, r.w_y, r.w_sum, r.M, r.W], g_scalar[f"sc_{tag}_wrs"][i])
        lid, pt, big_w = nls_sample(sp, cache, sc, R.stream(1, i, "light-select"))
        want = g_scalar[f"sc_{tag}_nls"][i]
        assert lid == int(want[0])
        np.testing.assert_array_equal(pt, want[1:4])
        assert big_w == pytest.approx(want[4], rel=RTOL)
        np.testing.assert_allclose(neural_di_shade(sp, cache, sc), g_scalar[f"sc_{tag}_ndi"][i], rtol=RTOL, atol=0)
        for j in range(k):
            assert unshadowed_weight(sp, j, sc) == pytest.approx(g_scalar[f"sc_{tag}_uw"][i, j], rel=RTOL, abs=0)
            np.testing.assert_allclose(unshadowed_rgb_one(sp, j, sc), g_scalar[f"sc_{tag}_urgb"][i, j],
                                       rtol=RTOL, atol=0)
    ctx = PixelCtx(sc, pos, nrm, alb)
    np.testing.assert_allclose(ctx.phat_ids(g_scalar[f"sc_{tag}_phat_ids"]), g_scalar[f"sc_{tag}_phat"],
                               rtol=RTOL, atol=0)


def test_wrs_select_validation():
    with pytest.raises(ValueError):
        wrs_select(np.zeros((2, 2)), R.stream(0))
    with pytest.raises(ValueError):
        wrs_select([0.5, -1.0], R.stream(0))
    r = wrs_select([0.0, 0.0], R.stream(0))
    assert r.empty and r.M == 2
