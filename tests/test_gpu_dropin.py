"""The drop-in boundary, exercised end to end through the reference itself.

baseline/_ref holds the UNMODIFIED reference package (tools/install_reference.sh;
it travels to the GPU box).  These tests run the reference's own frame loop
(``viscache.render.render_frame``, render.py:283-375) with ``dropin.install()``
rebinding its hot-path names to the CUDA versions, and compare frame by frame
with the same loop run purely on the reference's CPU code.  Then they run the
reference's own test modules through the ``nvc_inject`` pytest plugin.
"""

import dataclasses
import os
import subprocess
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)
if not os.path.isdir(os.path.join(REF, "viscache")):
    pytest.skip("baseline/_ref (the reference install, tools/install_reference.sh) is absent",
                allow_module_level=True)

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nvc_numba_cache")
sys.path.insert(0, REF)
import importlib  # noqa: E402

VR = importlib.import_module("viscache.render")   # the reference (the package re-exports a render() function)
from viscache.scene import scene_from_dict as ref_scene  # noqa: E402
from viscache.scenes import boxes_scene as ref_boxes  # noqa: E402

from paper_2506_05930_b200 import PRECISION_FP16, PRECISION_FP32, VisibilityCache, _lib, dropin  # noqa: E402


def run_frames(mode, frames, scene, cam, **cfg):
    st = VR.FrameState(scene, VR.RenderConfig(mode=mode, seed=3, frames=frames, **cfg), camera=cam)
    out = []
    for _ in range(frames):
        VR.render_frame(scene, st)
        out.append((st.last_estimate.copy(), st.last_loss))
    return st, out


def fresh_scene(w=96, h=54):
    s = ref_scene(ref_boxes(8))
    return s, dataclasses.replace(s.camera, width=w, height=h)


@pytest.fixture(scope="module")
def cpu_runs():
    """The reference loop on its own CPU code (no injection)."""
    assert not dropin.installed()
    runs = {}
    for mode in (VR.MODE_NLS, VR.MODE_NEURAL_DI, VR.MODE_CNVC, VR.MODE_RIS, VR.MODE_RESTIR, VR.MODE_CNVC_RESTIR):
        s, cam = fresh_scene()
        runs[mode] = run_frames(mode, 3, s, cam)[1]
    return runs


@pytest.mark.parametrize("precision", [PRECISION_FP32, PRECISION_FP16])
@pytest.mark.parametrize("mode", ["nls", "neural-di", "cnvc", "ris", "restir", "cnvc-restir"])
def test_reference_render_frame_on_the_cuda_cache(cpu_runs, mode, precision):
    """render_frame passes (1) G-buffer, (2)-(3) train_frame, (4) NLS / Neural DI /
    clustered sampling / RIS / ReSTIR (temporal-first: RIS or C-NVC initial
    reservoirs, temporal then spatial reuse), (5) shade_batch through the
    injected names.  Per frame:
    the training loss within 1e-2 of the reference's (SURVEY 8(c) band), and the
    image: on the f32 parity path nearly every pixel's estimate matching and
    the frame mean within 1e-3; on the fp16 tcgen05 path (visibility within
    4e-3) the frame mean within 1 %."""
    s, cam = fresh_scene()
    dropin.install(precision=precision)
    try:
        st, got = run_frames(mode, 3, s, cam)
        if mode in VR.NEURAL_MODES:
            assert isinstance(st.cache, VisibilityCache) and st.cache.precision == precision
        if mode in VR.RESTIR_MODES:
            from paper_2506_05930_b200.restir import ReservoirGrid
            assert isinstance(st.prev, ReservoirGrid)          # the reservoirs stayed on the device
    finally:
        dropin.uninstall()
    want = cpu_runs[mode]
    for f, ((est, loss), (rest, rloss)) in enumerate(zip(got, want)):
        assert (loss is None and rloss is None) or loss == pytest.approx(rloss, rel=1e-2), (mode, f)
        # a pixel "matches" when its estimate agrees to 1e-4: the same light choice
        # and point (a different choice moves it by O(1)); W = w_sum / w_sel still
        # carries the visibility, which the f32 train steps leave ~1e-7 apart, and
        # the f64 restatement of the numba factor kernel (acos, ~1e-10)
        rtol = 1e-4
        same = np.mean(np.all(np.isclose(est, rest, rtol=rtol, atol=1e-12), axis=1))
        mean_rel = abs(est.mean() - rest.mean()) / rest.mean()
        print(f"{mode} prec {precision} frame {f}: loss {loss} (ref {rloss}), identical pixels "
              f"{same:.4f}, frame-mean rel diff {mean_rel:.2e}")
        if precision == PRECISION_FP32:
            assert same > 0.99 and mean_rel < 1e-3, (mode, f, same, mean_rel)
        else:   # fp16 visibilities move choices where u*s_k sits within ~4e-3 of w_k
            assert same > 0.4 and mean_rel < 1e-2, (mode, f, same, mean_rel)


def test_reference_types_accepted_directly():
    """The reference's own PixelCtx / GBuffer / ClusterSet / configs go straight
    into this package's functions (no conversion by the caller)."""
    from viscache.cache import MODE_LIGHTS
    from viscache.sampling import PixelCtx as RefCtx
    from viscache.training import TrainFrameConfig as RefTF
    from paper_2506_05930_b200 import make_cache, nls_sample_batch, train_frame
    from paper_2506_05930_b200 import rng as R
    s, cam = fresh_scene(40, 24)
    gb = VR.make_gbuffer(s, cam)
    rctx = RefCtx(s, gb.flat("position"), gb.flat("normal"), gb.flat("albedo"))
    c = make_cache(s, MODE_LIGHTS, seed=1, precision=PRECISION_FP32)
    loss = train_frame(s, cam, c, RefTF(n_world=512, n_screen=512, seed=1), frame=0)
    assert 0.0 < loss < 1.0
    ids, pts, w = nls_sample_batch(rctx, c, R.stream(1, 0, "light-select"))
    assert ids.shape == (rctx.n,) and pts.shape == (rctx.n, 3) and np.all(w[ids >= 0] > 0)
    # the same pixels through this package's own context give identical choices
    from paper_2506_05930_b200 import PixelCtx
    mine = PixelCtx(s, rctx.positions, rctx.normals, rctx.albedos)
    ids2, _, _ = nls_sample_batch(mine, c, R.stream(1, 0, "light-select"))
    np.testing.assert_array_equal(ids, ids2)


def test_write_through_params_and_adam():
    """grid_params / net_params are live views like the reference's arrays
    (cache.py:41-48): writes reach the device, updates reach held views."""
    from viscache.cache import MODE_LIGHTS
    from paper_2506_05930_b200 import make_cache
    s, cam = fresh_scene(40, 24)
    c = make_cache(s, MODE_LIGHTS, seed=2, precision=PRECISION_FP32)
    for w in c.net_params.weights:
        w[:] = 0
    for b in c.net_params.biases:
        b[:] = 0
    pos = np.random.default_rng(0).uniform(s.aabb_min, s.aabb_max, (300, 3))
    np.testing.assert_array_equal(c.infer(pos), 0.5)                # sigmoid(0)
    c = make_cache(s, MODE_LIGHTS, seed=2, precision=PRECISION_FP32)   # non-zero weights: the grid gets gradients
    grid = c.grid_params                                            # held view
    before = grid.copy()
    c.train_step(pos, np.ones((300, c.output_dim), np.float32))
    assert not np.array_equal(grid, before)                         # Adam's update reached the view
    np.testing.assert_array_equal(grid, c.params[:grid.size].cpu().numpy().reshape(grid.shape))
    st = c.adam
    assert st.t == 1 and set(st.m) == {"grid", "w0", "b0", "w1", "b1", "w2", "b2"}
    assert np.abs(st.m["w2"]).max() > 0
    with pytest.raises(ValueError, match="float32 master"):
        make_cache(s, MODE_LIGHTS, dtype=np.float64)


@pytest.mark.parametrize("module", ["test_sampling.py", "test_training.py", "test_mlp.py", "test_render.py"])
def test_reference_suite_through_the_plugin(module):
    """The reference's own tests with the CUDA cache injected (tests/nvc_inject.py).
    Allowed failures: those the reference itself fails in this image (shapely
    absent: 2 analytic-penumbra tests; 1 NRC-vs-NLS test that fails on the
    reference's own CPU path too) and one test that spies on a CPU-internal
    function the device path replaces."""
    allowed = {"test_penumbra_mean_matches_analytic_fraction", "test_converged_prediction_matches_mean_visibility",
               "test_blurrier_than_neural_di_on_shadow_boundary",
               # spies on the reference's CPU visibility_batch (training.py internals); the
               # device path computes the same batch x lights labels without calling it
               "test_shadow_ray_budget_is_batch_times_lights"}
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.join(ROOT, "tests"), ROOT, REF]),
               NVC_INJECT_PRECISION="fp32")
    r = subprocess.run([sys.executable, "-m", "pytest", "-p", "nvc_inject", "-p", "no:cacheprovider", "-q",
                        "-rf", "--rootdir", os.path.join(REF, "viscache_tests"),
                        os.path.join(REF, "viscache_tests", module)],
                       cwd=os.path.join(REF, "viscache_tests"), env=env, capture_output=True, text=True, timeout=1800)
    tail = r.stdout[-3000:]
    print(tail)
    failed = {line.split("::")[-1].split(" ")[0] for line in r.stdout.splitlines() if line.startswith("FAILED")}
    assert "nvc_inject: reference names rebound" in r.stdout
    assert failed <= allowed, tail
    assert " passed" in tail
