"""Parity at the headline configurations (BASELINE configs[1] = C2, configs[3] = C4).

* C2 loss curve over the 60 online frames of configs[1] against the reference's
  own float32 and float64 runs (tests/golden/curves.npz, make_golden.py
  gen_long_curves), and C4 (3x128 MLP, K=128) over 8 frames.
* Inference at trained scale: a reference-trained C1 cache (its parameters are
  in the fixture) through the fp32 and the fp16/tcgen05 paths against the
  reference's own outputs; the GPU-trained C2 cache against the oracle on the
  same parameters.
* fp16 encoder features (the perf path's k_enc_tiles2 tiles) against the oracle
  with a per-element rounding bound.
* How often the f32 luminance table changes a C2 light choice against the
  reference's f64 table on identical visibilities.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from oracle import vc_oracle as O  # noqa: E402
from paper_2506_05930_b200 import (PRECISION_FP16, PRECISION_FP32, HashGridConfig, MLPParams,  # noqa: E402
                                   MODE_LIGHTS, VisibilityCache, gbuffer_and_ctx, scene_from_dict,
                                   train_frame, TrainFrameConfig)
from paper_2506_05930_b200 import rng as R  # noqa: E402
from paper_2506_05930_b200 import _lib  # noqa: E402
from paper_2506_05930_b200.sampling import nls_sample_device  # noqa: E402
from paper_2506_05930_b200.scenes import boxes_point_scene, boxes_scene, rooms_scene  # noqa: E402

from conftest import golden  # noqa: E402

U16 = 2.0 ** -11          # fp16 unit roundoff
FP16_VIS_TOL = 4e-3       # stated fp16 visibility tolerance
LOSS_RTOL = 1e-2          # per-frame loss band: reference f32 vs f64 reaches 3.1e-3 at C2


@pytest.fixture(scope="module")
def g_curves():
    return golden("curves")


def grid_cfg(scene, levels, tsize):
    return HashGridConfig(levels=levels, table_size=tsize, features_per_level=2,
                          aabb_min=scene.aabb_min, aabb_max=scene.aabb_max)


def oracle_of(cache, scene, levels, tsize, hidden):
    oc = O.Cache(O.Grid(levels=levels, features_per_level=2, table_size=tsize, aabb_min=scene.aabb_min,
                        aabb_max=scene.aabb_max), cache.output_dim, hidden=hidden)
    oc.unflat(cache.params.cpu().numpy())
    return oc


def umma_off(r, k, rows, kp):
    """common.cuh umma_off: byte offset of (row r, column k) in a swizzled K-major fp16 tile."""
    lg = 7 if kp >= 64 else (6 if kp == 32 else 5)
    kb = 2 * k
    atom, within = kb >> lg, kb & ((1 << lg) - 1)
    cs = (within >> 4) ^ ((r & 7) >> (7 - lg))
    return (atom * rows << lg) + (r << lg) + (cs << 4) + (within & 15)


def perf_features(cache, pos):
    """Run the query front end (k_enc_tiles2 + MLP) and read the fp16 feature
    tiles it left in the workspace back as a (n, L*F) float array."""
    n = pos.shape[0]
    g = cache.grid_cfg
    kf = g.levels * g.features_per_level
    kp = 16 if kf <= 16 else (32 if kf <= 32 else (kf + 63) // 64 * 64)
    pt = torch.from_numpy(pos).to(cache.device)
    ws = cache.query_workspace(n)
    _lib.call("nvc_query_front", cache.model, pt.data_ptr(), n, _lib.ptr(ws), _lib.stream_ptr())
    torch.cuda.synchronize()
    ntiles = (n + 127) // 128
    raw = ws[:ntiles * 128 * kp * 2].cpu().numpy().view(np.uint8)
    p = np.arange(n)[:, None]
    k = np.arange(kf)[None, :]
    off = (p // 128) * (128 * kp * 2) + umma_off(p % 128, k, 128, kp)
    lo, hi = raw[off].astype(np.uint16), raw[off + 1].astype(np.uint16)
    return (lo | (hi << 8)).view(np.float16).astype(np.float64)


# ---------------------------------------------------------------------------
# fp16 encoder features
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("variant", ["tiles2", "NVC_ENC_F32"])
@pytest.mark.parametrize("levels,tsize", [(16, 1 << 19), (8, 1 << 14)])
def test_fp16_features_within_rounding_bound(monkeypatch, variant, levels, tsize):
    """Perf-path features = sum_c h(w_c) h(t_c) accumulated in f32, rounded to
    fp16 once (h = round to fp16).  Against the f32 oracle blend, per element:
        |d| <= 2u * sum_c w_c |t_c| + u |f| + 2^-24 * sum_c |t_c| + 1e-7
    (u = 2^-11: table rounding + weight rounding, final store, fp16 subnormal
    weights; the f32 accumulation error is far below the slack).  Trained-scale
    N(0, 0.3) tables, C2 and C1 grids, random and G-buffer positions."""
    if variant != "tiles2":
        monkeypatch.setenv(variant, "1")
    scene = scene_from_dict(boxes_scene(32))
    c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(scene, levels, tsize), seed=0, hidden_dims=(64, 64, 64))
    g = np.random.default_rng(11)
    table = (g.standard_normal(c.grid_params.shape) * 0.3).astype(np.float32)
    c.grid_params = table
    _, ctx = gbuffer_and_ctx(scene, scene.camera.resized(160, 90))
    pos = np.concatenate([g.uniform(scene.aabb_min, scene.aabb_max, (20000, 3)), ctx.positions])
    got = perf_features(c, pos)
    og = O.Grid(levels=levels, features_per_level=2, table_size=tsize, aabb_min=scene.aabb_min,
                aabb_max=scene.aabb_max)
    want, octx = O.encode(og, table, pos)
    want = want.astype(np.float64)
    s_w = np.zeros_like(want)
    s_abs = np.zeros_like(want)
    for lvl, (idx, w) in enumerate(octx):
        t = np.abs(table[lvl][idx].astype(np.float64))          # (n, 8, F)
        s_w[:, 2 * lvl:2 * lvl + 2] = (w[:, :, None] * t).sum(1)
        s_abs[:, 2 * lvl:2 * lvl + 2] = t.sum(1)
    bound = 2 * U16 * s_w + U16 * np.abs(want) + 2.0 ** -24 * s_abs + 1e-7
    err = np.abs(got - want)
    worst = np.argmax(err / bound)
    assert np.all(err <= bound), (err.flat[worst], bound.flat[worst])
    print(f"fp16 features: max |d| {err.max():.3e}, mean {err.mean():.3e}, "
          f"max |d|/bound {float((err / bound).max()):.3f}")


# ---------------------------------------------------------------------------
# inference at trained scale: reference-trained C1 cache
# ---------------------------------------------------------------------------
def test_reference_trained_c1_inference(g_curves):
    """The reference trained a C1 cache for 20 frames; its parameters and its
    outputs on 4096 random probes + every G-buffer hit are in the fixture.
    fp32 SIMT path: within 2e-6 (sgemm order); fp16/tcgen05 path: within the
    stated 4e-3."""
    scene = scene_from_dict(boxes_point_scene(8))
    c = VisibilityCache(MODE_LIGHTS, 8, grid_cfg(scene, 8, 1 << 14), seed=0, hidden_dims=(64, 64))
    ws = [g_curves[f"c1t_w{i}"] for i in range(3)]
    bs = [g_curves[f"c1t_b{i}"] for i in range(3)]
    c._upload(g_curves["c1t_grid"], MLPParams(ws, bs))
    pos, want = g_curves["c1t_probe_pos"], g_curves["c1t_probe_vis"]
    assert want.std() > 0.1            # genuinely trained: outputs span (0, 1)
    got32 = c.infer(pos, precision=PRECISION_FP32)
    np.testing.assert_allclose(got32, want, rtol=0, atol=2e-6)
    got16 = c.infer(pos, precision=PRECISION_FP16)
    d = np.abs(got16 - want)
    print(f"C1 reference-trained fp16 vis: max |d| {d.max():.3e}, mean {d.mean():.3e}")
    assert d.max() < FP16_VIS_TOL


# ---------------------------------------------------------------------------
# C2: 60-frame loss curve, trained-scale inference, f32-lum choice mismatch
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def c2_trained():
    scene = scene_from_dict(boxes_scene(32))
    c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(scene, 16, 1 << 19), seed=0, hidden_dims=(64, 64, 64))
    cfg = TrainFrameConfig()
    losses = np.array([train_frame(scene, scene.camera, c, cfg, frame=f) for f in range(60)])
    return scene, c, losses


def test_c2_loss_curve_60_frames(c2_trained, g_curves):
    """BASELINE configs[1]: 60 online frames of boxes32 at L=16 T=2^19 F=2, MLP
    3x64, K=32, 8192-sample batches.  Reference f32 vs f64 differ by up to
    3.1e-3 (rel) over these frames; the GPU curve stays within 1e-2 of both at
    every frame and its mean deviation stays at the f32/f64 noise level."""
    _, _, got = c2_trained
    ref32, ref64 = g_curves["c2_loss60_f32"], g_curves["c2_loss60_f64"]
    rel32, rel64 = np.abs(got - ref32) / ref32, np.abs(got - ref64) / ref64
    spread = np.abs(ref32 - ref64) / ref64
    print(f"C2 60 frames: max rel vs ref f32 {rel32.max():.2e} (mean {rel32.mean():.2e}), vs f64 "
          f"{rel64.max():.2e}; ref f32/f64 spread max {spread.max():.2e} (mean {spread.mean():.2e}); "
          f"loss {got[0]:.5f} -> {got[-1]:.5f} (ref {ref32[-1]:.5f})")
    assert rel32.max() < LOSS_RTOL and rel64.max() < LOSS_RTOL
    assert rel64.mean() < 3 * max(spread.mean(), 1e-3)
    assert got[-1] < 0.2 * got[0]        # it learned


def test_c2_loss_curve_60_frames_tensor_core_training(g_curves, monkeypatch):
    """The same 60 C2 frames with the training step on the tensor cores
    (k_train_tc: tcgen05 forward + backward, split bf16 operands ~17 bits, fp32
    TMEM accumulators).  The curve tracks the reference to 1e-3 over the first
    10 frames; from frame 11 (the first loss spike at lr 0.05) any trajectory
    whose GEMM arithmetic is not bit-faithful fp32 leaves the 1e-2 band --
    the fp32 step with its weights rounded to 23 bits does too
    (tools/precision_study.py, profiles/r2_precision_study.txt) -- which is why
    the fp32 SIMT step stays the default.  What is asserted beyond frame 10 is
    that it learns as well: the mean loss over frames 40-59 within 8 % of the
    reference's (perturbed fp32 runs: -1 % to +5 %; this step: ~+5 %)."""
    monkeypatch.setenv("NVC_TRAIN_TC", "1")
    scene = scene_from_dict(boxes_scene(32))
    c = VisibilityCache(MODE_LIGHTS, 32, grid_cfg(scene, 16, 1 << 19), seed=0, hidden_dims=(64, 64, 64))
    got = np.array([train_frame(scene, scene.camera, c, TrainFrameConfig(), frame=f) for f in range(60)])
    ref32, ref64 = g_curves["c2_loss60_f32"], g_curves["c2_loss60_f64"]
    rel32, rel64 = np.abs(got - ref32) / ref32, np.abs(got - ref64) / ref64
    print(f"C2 60 frames (tensor-core training): max rel vs ref f32 {rel32.max():.2e} (mean {rel32.mean():.2e}), "
          f"vs f64 {rel64.max():.2e}; loss {got[0]:.5f} -> {got[-1]:.5f}")
    assert rel32[:10].max() < 1e-3 and rel64[:10].max() < 1e-3
    late = got[40:].mean() / ref32[40:].mean() - 1.0
    print(f"frames 40-59 mean loss {got[40:].mean():.5f} vs ref {ref32[40:].mean():.5f} ({late:+.2%})")
    assert abs(late) < 0.08 and got[-1] < 0.2 * got[0]


def test_c2_trained_inference_vs_oracle(c2_trained, g_curves):
    """The GPU-trained C2 cache (60 frames) vs the oracle on the SAME parameters,
    at 4096 random probes and 1080p G-buffer pixels: fp32 path within 1e-5,
    fp16/tcgen05 path within the stated tolerance.  Also the mean-abs distance
    to the reference-trained cache's probe outputs, against the reference's own
    f32-vs-f64 distance (pointwise trained parameters diverge by design:
    SURVEY 8(c))."""
    scene, c, _ = c2_trained
    oc = oracle_of(c, scene, 16, 1 << 19, (64, 64, 64))
    _, ctx = gbuffer_and_ctx(scene, scene.camera.resized(1920, 1080))
    pix = ctx.positions[np.random.default_rng(3).choice(ctx.n, 32768, replace=False)]
    pos = np.concatenate([g_curves["c2_probe_pos"], pix])
    want = oc.infer(pos)
    assert want.std() > 0.1
    got32 = c.infer(pos, precision=PRECISION_FP32)
    np.testing.assert_allclose(got32, want, rtol=0, atol=1e-5)
    got16 = c.infer(pos, precision=PRECISION_FP16)
    d = np.abs(got16 - want)
    print(f"C2 trained (60 frames) fp16 vis vs oracle: max |d| {d.max():.3e}, mean {d.mean():.3e}, "
          f"p99.9 {np.quantile(d, 0.999):.3e}")
    assert d.max() < FP16_VIS_TOL and d.mean() < 2e-4
    probe = g_curves["c2_probe_pos"]
    mine = c.infer(probe, precision=PRECISION_FP32)
    ref32, ref64 = g_curves["c2_probe_vis_f32"], g_curves["c2_probe_vis_f64"]
    m_ref, m_me = np.abs(ref32 - ref64).mean(), np.abs(mine - ref32).mean()
    print(f"C2 trained probes: mean |GPU - ref f32| {m_me:.2e}; ref f32 vs f64 {m_ref:.2e}")
    assert m_me < 3 * m_ref


def test_c2_f32_lum_choice_mismatch(c2_trained):
    """The perf path's f32 luminance table against the reference's f64 one on
    the same visibilities (trained C2 cache, 1080p frame): the fraction of
    pixels whose light choice differs is reported and bounded; the f64 table is
    bit-exact to the reference by construction (test_gpu_parity)."""
    scene, c, _ = c2_trained
    from paper_2506_05930_b200.sampling import PixelCtx
    _, ctx32 = gbuffer_and_ctx(scene, scene.camera.resized(1920, 1080), table_dtype=np.float32)
    ctx64 = PixelCtx(scene, ctx32.pos, ctx32.nrm, ctx32.alb, table_dtype=np.float64)
    key = R.stream_key(0, 0, "light-select")
    i32, p32, w32 = nls_sample_device(ctx32, c, key)
    i64, p64, w64 = nls_sample_device(ctx64, c, key)
    torch.cuda.synchronize()
    live = (i64 >= 0).sum().item()
    diff = (i32 != i64).sum().item()
    rate = diff / ctx32.n
    relw = ((w32 - w64).abs() / w64.abs().clamp_min(1e-300))[(i32 == i64) & (i64 >= 0)]
    print(f"C2 f32-lum light-choice mismatch: {diff} of {ctx32.n} pixels ({rate:.2e}; {live} live); "
          f"W rel diff on agreeing pixels max {relw.max().item():.2e}")
    assert rate < 1e-4


# ---------------------------------------------------------------------------
# C4: 3x128 MLP, K=128 lights
# ---------------------------------------------------------------------------
def test_c4_loss_curve(g_curves):
    """BASELINE configs[3]: rooms128 (K=128), L=16 T=2^19, MLP 3x128, 8 frames
    against the reference's f32 and f64 runs (which agree to 4e-6)."""
    scene = scene_from_dict(rooms_scene(128))
    c = VisibilityCache(MODE_LIGHTS, 128, grid_cfg(scene, 16, 1 << 19), seed=0, hidden_dims=(128, 128, 128))
    cfg = TrainFrameConfig()
    got = np.array([train_frame(scene, scene.camera, c, cfg, frame=f) for f in range(8)])
    ref32, ref64 = g_curves["c4_loss_f32"], g_curves["c4_loss_f64"]
    rel = np.abs(got - ref64) / ref64
    print(f"C4 8 frames: max rel vs ref f64 {rel.max():.2e}; loss {got[0]:.5f} -> {got[-1]:.5f}")
    assert np.max(np.abs(got - ref32) / ref32) < LOSS_RTOL and rel.max() < LOSS_RTOL
