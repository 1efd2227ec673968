"""RIS / screen-space ReSTIR baselines on the GPU (reference sampling.py:369-637)
against the reference's own outputs (tests/golden/restir.npz, make_golden.py
gen_restir) on boxes8 at 48x32.

Bit-exact: candidate ids (integers() with a kept 32-bit half from an earlier
integers() call on the same stream), selected lights, emitter points, M, the
validity flags and the stream continuation.  Target weights come from the
device FP64 factor table (~1e-12 from numba's), so w_y / w_sum / W are held
to 1e-9 relative."""

import types

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2506_05930_b200 import (MODE_LIGHTS, PixelCtx, gbuffer_and_ctx, kmeans_cluster,  # noqa: E402
                                   scene_from_dict)
from paper_2506_05930_b200 import rng as R  # noqa: E402
from paper_2506_05930_b200.restir import (ReservoirGrid, cnvc_initial_batch, restir_spatial_batch,  # noqa: E402
                                          restir_temporal_batch, ris_initial_batch)
from paper_2506_05930_b200.scenes import boxes_scene  # noqa: E402

from conftest import golden  # noqa: E402

FIELDS = ("y", "point", "w_y", "w_sum", "M", "W", "valid")


class WaveCache:
    mode = MODE_LIGHTS

    def __init__(self, k):
        self.output_dim = k

    def infer(self, positions):
        pos = np.atleast_2d(np.asarray(positions, np.float64))
        ph = pos @ np.array([1.3, 2.1, 0.7])
        return (0.5 + 0.4 * np.sin(ph[:, None] + np.arange(self.output_dim))).astype(np.float32)


@pytest.fixture(scope="module")
def g():
    return golden("restir")


@pytest.fixture(scope="module")
def frame():
    s = scene_from_dict(boxes_scene(8))
    gb, ctx = gbuffer_and_ctx(s, s.camera.resized(48, 32))
    return s, gb, ctx


def check(grid, g, tag, rng=None):
    for k in ("y", "M", "valid", "point"):
        np.testing.assert_array_equal(getattr(grid, k), g[f"{tag}_{k}"], err_msg=f"{tag}.{k}")
    for k in ("w_y", "w_sum", "W"):
        np.testing.assert_allclose(getattr(grid, k), g[f"{tag}_{k}"], rtol=1e-9, atol=0, err_msg=f"{tag}.{k}")
    if rng is not None:
        np.testing.assert_array_equal(rng.random(3), g[f"{tag}_next"], err_msg=f"{tag}: stream continuation")


def grid_from(g, tag):
    return types.SimpleNamespace(**{k: np.array(g[f"{tag}_{k}"]) for k in FIELDS})


def test_ris_initial(g, frame):
    _, _, ctx = frame
    r0 = R.stream(0, 0, "restir-initial")
    np.testing.assert_array_equal(r0.integers(0, 7, size=3), g["pre_ints"])     # leaves a kept 32-bit half
    check(ris_initial_batch(ctx, r0, 8), g, "ris0", r0)
    r1 = R.stream(0, 1, "restir-initial")
    check(ris_initial_batch(ctx, r1, 8), g, "ris1", r1)


def test_temporal_both_clamp_modes(g, frame):
    _, _, ctx = frame
    cur, prev = grid_from(g, "ris1"), grid_from(g, "ris0")
    rt = R.stream(0, 1, "restir-temporal")
    check(restir_temporal_batch(cur, prev, ctx, rt, 20.0, "m"), g, "tm", rt)
    prev.valid[::3] = False
    prev.M[1::5] = 60.0
    rt2 = R.stream(0, 2, "restir-temporal")
    check(restir_temporal_batch(cur, prev, ctx, rt2, 2.0, "contribution"), g, "tc", rt2)
    rt3 = R.stream(0, 3, "restir-temporal")
    check(restir_temporal_batch(ReservoirGrid.of(cur, ctx.device), ReservoirGrid.of(prev, ctx.device), ctx, rt3,
                                2.0, "m"), g, "tm2", rt3)
    with pytest.raises(ValueError):
        restir_temporal_batch(cur, prev, ctx, R.stream(0), 2.0, "bogus")


@pytest.mark.parametrize("rad", [32, 4])
def test_spatial(g, frame, rad):
    _, gb, ctx = frame
    rs = R.stream(0, rad, "restir-spatial")
    out = restir_spatial_batch(grid_from(g, "tm"), ctx, gb.shape, gb.flat("hit"), gb.flat("depth"), ctx.normals,
                               rs, rad, 4)
    check(out, g, f"sp{rad}", rs)


def test_cnvc_initial(g, frame):
    s, _, ctx = frame
    cl = kmeans_cluster(s.lights, 4, R.stream(0, "clustering"))
    rc = R.stream(0, 2, "restir-initial")
    check(cnvc_initial_batch(ctx, WaveCache(4), cl, rc), g, "cn", rc)


def test_chain_on_device_full_hd():
    """The render_frame chain (RIS -> temporal -> spatial) stays on the device at
    1080p and keeps the reservoir invariant W = w_sum / (M * w_y)."""
    s = scene_from_dict(boxes_scene(32))
    gb, ctx = gbuffer_and_ctx(s, s.camera.resized(1920, 1080))
    g0 = ris_initial_batch(ctx, R.stream(0, 0, "restir-initial"), 8)
    g1 = ris_initial_batch(ctx, R.stream(0, 1, "restir-initial"), 8)
    t = restir_temporal_batch(g1, g0, ctx, R.stream(0, 1, "restir-temporal"))
    sp = restir_spatial_batch(t, ctx, gb.shape, ctx.hit, gb.flat("depth"), ctx.nrm, R.stream(0, 1, "restir-spatial"))
    y, W, ws, M, wy = (sp.d[k] for k in ("y", "W", "w_sum", "M", "w_y"))
    live = y >= 0
    assert live.float().mean().item() > 0.3
    torch.testing.assert_close(W[live], ws[live] / (M[live] * wy[live]), rtol=1e-15, atol=0)
    assert (M[live] >= 16).all()
