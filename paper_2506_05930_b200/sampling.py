"""Light selection driven by the cache: drop-in for ``viscache.sampling``
(sampling.py:19-222: WRS, unshadowed weights, NLS, Neural DI).

Every function keeps the reference signature and numpy outputs.  The work
runs on the GPU: the fused ``nvc_nls_sample`` / ``nvc_neural_di`` kernels when
the cache is this package's :class:`VisibilityCache`, otherwise (any
duck-typed cache exposing ``infer``, e.g. the reference tests' FixedCache)
``cache.infer`` supplies the visibilities and ``nvc_nls_from_vis`` does the
selection.  Uniforms come from the caller's Philox stream by global draw
index, so results are bit-identical to the reference given the same weights,
and screen-tile shards (``p_first``/``p_total``) reproduce the whole frame.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import rng as rngmod
from .scene import LUMA, device_scene

CLAMP_FLOOR = 0.001


def clamp_visibility(v, floor: float = CLAMP_FLOOR):
    return np.maximum(v, floor)


@dataclass
class ShadingPoint:
    position: np.ndarray
    normal: np.ndarray
    albedo: np.ndarray
    omega_o: np.ndarray | None = None

    def __post_init__(self):
        self.position = np.asarray(self.position, dtype=np.float64)
        self.normal = np.asarray(self.normal, dtype=np.float64)
        self.albedo = np.asarray(self.albedo, dtype=np.float64)


@dataclass
class Reservoir:
    """Invariant (nonempty): W == w_sum / (M * w_y)  (sampling.py:46-62)."""

    y: int = -1
    point: np.ndarray | None = None
    w_y: float = 0.0
    w_sum: float = 0.0
    M: float = 0.0
    W: float = 0.0

    @property
    def empty(self) -> bool:
        return self.y < 0 or self.W <= 0.0


def _dev(a, torch, device, dtype):
    if isinstance(a, torch.Tensor):
        return a.to(device, dtype).contiguous()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64 if dtype == torch.float64 else np.float32)).to(device)


def wrs_select_batch(weights, rng):
    """Row-wise streaming WRS on the GPU; (index, w_selected, w_sum), index -1 for all-zero rows."""
    torch = _lib.require_cuda()
    w = np.atleast_2d(np.asarray(weights, dtype=np.float64))
    p, k = w.shape
    key, off = rngmod.position(rng)
    dev = torch.device("cuda", torch.cuda.current_device())
    wd = _dev(w, torch, dev, torch.float64)
    idx = torch.empty(p, dtype=torch.int64, device=dev)
    wsel = torch.empty(p, dtype=torch.float64, device=dev)
    wsum = torch.empty(p, dtype=torch.float64, device=dev)
    _lib.call("nvc_wrs_select", wd.data_ptr(), p, k, key, off, idx.data_ptr(), wsel.data_ptr(),
              wsum.data_ptr(), _lib.stream_ptr())
    rngmod.advance(rng, p * k)
    return idx.cpu().numpy(), wsel.cpu().numpy(), wsum.cpu().numpy()


def wrs_select(weights, rng) -> Reservoir:
    w = np.asarray(weights, dtype=np.float64)
    if w.ndim != 1 or w.size < 1:
        raise ValueError("weight stream must be a nonempty 1-d sequence")
    if np.any(w < 0):
        raise ValueError("weights must be nonnegative")
    idx, w_sel, w_sum = wrs_select_batch(w[None, :], rng)
    if idx[0] < 0:
        return Reservoir(M=w.size)
    return Reservoir(y=int(idx[0]), w_y=float(w_sel[0]), w_sum=float(w_sum[0]), M=w.size,
                     W=float(w_sum[0] / (w.size * w_sel[0])))


class PixelCtx:
    """Per-pixel shading data resident on the GPU, with lazily built
    light-major (K, P) factor / luminance tables (sampling.py:109-160).

    ``table_dtype`` float64 (default: the reference's FP64 tables, so light
    choices are bit-exact given the visibilities) or float32 (half the hot
    loop's table traffic; the perf path requests it explicitly -- its choice
    mismatch rate against f64 is measured in tests/test_gpu_headline.py)."""

    def __init__(self, scene, positions, normals, albedos, factors=None, table_dtype=np.float64,
                 device=None):
        torch = _lib.require_cuda()
        self.scene = scene
        self.dscene = device_scene(scene, device)
        dev = self.dscene.device
        self.device = dev
        self.pos = _dev(np.atleast_2d(positions) if not isinstance(positions, torch.Tensor) else positions,
                        torch, dev, torch.float64).reshape(-1, 3)
        self.nrm = _dev(np.atleast_2d(normals) if not isinstance(normals, torch.Tensor) else normals,
                        torch, dev, torch.float64).reshape(-1, 3)
        self.alb = _dev(np.atleast_2d(albedos) if not isinstance(albedos, torch.Tensor) else albedos,
                        torch, dev, torch.float64).reshape(-1, 3)
        self._host_pos = None if isinstance(positions, torch.Tensor) else np.ascontiguousarray(
            np.atleast_2d(positions), dtype=np.float64)
        self.table_dtype = np.dtype(table_dtype)
        self._tdt = torch.float64 if self.table_dtype == np.float64 else torch.float32
        self._factor = None
        self._lum = None
        self._masks = {}
        if factors is not None:
            self._factor = _dev(np.asarray(factors).T, torch, dev, self._tdt).contiguous()

    @property
    def n(self) -> int:
        return self.pos.shape[0]

    @property
    def positions(self) -> np.ndarray:
        if self._host_pos is None:
            self._host_pos = self.pos.cpu().numpy()
        return self._host_pos

    @property
    def normals(self) -> np.ndarray:
        if getattr(self, "_host_nrm", None) is None:
            self._host_nrm = self.nrm.cpu().numpy()
        return self._host_nrm

    @property
    def albedos(self) -> np.ndarray:
        if getattr(self, "_host_alb", None) is None:
            self._host_alb = self.alb.cpu().numpy()
        return self._host_alb

    def _build(self, want_lum: bool) -> None:
        import torch
        k, p = self.dscene.n_lights, self.n
        fac = None if self._factor is not None else torch.empty((k, p), dtype=self._tdt, device=self.device)
        lum = torch.empty((k, p), dtype=self._tdt, device=self.device) if want_lum else None
        if fac is None and lum is None:
            return
        if fac is None:
            # factors supplied by the caller: lum = factor * (albedo . LUMA*L)/pi on device
            scale = (self.alb @ (torch.as_tensor(LUMA, device=self.device)[:, None]
                                 * self.dscene.lt_radiance.T)) / np.pi
            self._lum = (self._factor.to(torch.float64) * scale.T).to(self._tdt).contiguous()
            return
        _lib.call("nvc_light_factors", self.dscene.struct, self.pos.data_ptr(), self.nrm.data_ptr(),
                  self.alb.data_ptr(), p, p, int(self._tdt == torch.float64), fac.data_ptr(), _lib.ptr(lum),
                  _lib.stream_ptr())
        self._factor = fac
        if want_lum:
            self._lum = lum

    def factor_device(self):
        if self._factor is None:
            self._build(want_lum=self._lum is None)
        return self._factor

    def lum_device(self):
        if self._lum is None:
            self._build(want_lum=True)
        return self._lum

    def mask_device(self, which: str = "lum"):
        """Per-pixel nonzero bitmask of the lum/factor table: ceil(K/32) words per
        pixel, word-major (word w of pixel p at w * stride + p)."""
        import torch
        if which not in self._masks:
            t = self.lum_device() if which == "lum" else self.factor_device()
            words = (self.dscene.n_lights + 31) // 32
            m = torch.empty(words * t.shape[1], dtype=torch.int32, device=self.device)
            _lib.call("nvc_table_mask", t.data_ptr(), int(t.dtype == torch.float64), t.shape[1], self.n,
                      self.dscene.n_lights, m.data_ptr(), _lib.stream_ptr())
            self._masks[which] = m
        return self._masks[which]

    def factor_matrix(self) -> np.ndarray:
        """(P, K) f64 host copy of the factor table (memoized like the reference's)."""
        if getattr(self, "_host_fac", None) is None:
            self._host_fac = self.factor_device().T.to(dtype=__import__("torch").float64).cpu().numpy()
        return self._host_fac

    @property
    def _factors(self):
        """The reference PixelCtx's cached factor matrix (sampling.py:117), read by
        its ReSTIR/RIS code: the host table once built on the device, else None."""
        return self.factor_matrix() if self._factor is not None else None

    def lum_matrix(self) -> np.ndarray:
        """(P, K) f64 host copy of the luminance table (memoized)."""
        if getattr(self, "_host_lum", None) is None:
            self._host_lum = self.lum_device().T.to(dtype=__import__("torch").float64).cpu().numpy()
        return self._host_lum

    def phat_ids(self, ids) -> np.ndarray:
        """Luminance target weight of one light per pixel, id < 0 -> 0
        (sampling.py:141-155): f * (albedo . LUMA*L_e)/pi with the reference's
        per-row einsum, f from the device factor table (FP64 restatement of
        the numba factor kernel, within 1e-10 of it)."""
        ids = np.asarray(ids)
        safe = np.maximum(ids, 0)
        f = np.take_along_axis(self.factor_matrix(), safe[:, None], 1)[:, 0]
        rad = self.scene.lt_radiance[safe]
        scale = np.einsum("pc,pc->p", self.albedos, LUMA * rad) / np.pi
        return np.where(ids >= 0, f * scale, 0.0)

    def unshadowed_rgb(self, vis) -> np.ndarray:
        import torch
        v = _dev(np.asarray(vis, np.float64), torch, self.device, torch.float64)
        f = self.factor_device().to(torch.float64).T
        rgb = ((v * f) @ self.dscene.lt_radiance) * self.alb / np.pi
        return rgb.cpu().numpy()


def as_pixel_ctx(ctx) -> PixelCtx:
    """This package's PixelCtx for ``ctx``.  A foreign context -- the reference's
    ``viscache.sampling.PixelCtx`` or any object with ``scene``, ``positions``,
    ``normals``, ``albedos`` (and optionally precomputed ``_factors``) -- is
    wrapped once on the device (f64 tables, as the reference's) and the
    wrapper memoized on it, so a caller that keeps its context per camera
    (render.py:128-142) uploads it once."""
    if isinstance(ctx, PixelCtx):
        return ctx
    memo = getattr(ctx, "__dict__", {}).get("_nvc_ctx")
    if memo is not None and memo[0] == ctx.positions.ctypes.data:
        return memo[1]
    factors = getattr(ctx, "_factors", None)
    mine = PixelCtx(ctx.scene, ctx.positions, ctx.normals, ctx.albedos, factors=factors, table_dtype=np.float64)
    if hasattr(ctx, "__dict__"):
        ctx.__dict__["_nvc_ctx"] = (ctx.positions.ctypes.data, mine)
    return mine


def _ctx_for(sp: ShadingPoint, scene) -> PixelCtx:
    return PixelCtx(scene, sp.position[None, :], sp.normal[None, :], sp.albedo[None, :],
                    table_dtype=np.float64)


def unshadowed_weight(sp: ShadingPoint, light_id: int, scene) -> float:
    return float(_ctx_for(sp, scene).phat_ids(np.array([light_id]))[0])


def unshadowed_rgb_one(sp: ShadingPoint, light_id: int, scene) -> np.ndarray:
    f = _ctx_for(sp, scene).factor_matrix()[0, light_id]
    return sp.albedo / np.pi * scene.lt_radiance[light_id] * f


def _is_native(cache) -> bool:
    from .cache import VisibilityCache
    return isinstance(cache, VisibilityCache)


FACTOR_CACHE_LIMIT = 64_000_000     # render.py:46


def _fused(cache) -> bool:
    """This package's cache on its fp16 tcgen05 query path: the fused
    encode -> MLP -> selection kernels.  A cache set to PRECISION_FP32 (the
    parity path) or a foreign cache gives its visibilities first."""
    from .cache import PRECISION_FP16
    return _is_native(cache) and cache.precision == PRECISION_FP16


def _visibility_device(ctx, cache):
    """(P, K) f32 CUDA visibilities of ctx's pixels from any cache."""
    import torch
    if _is_native(cache):
        return cache.infer_device(ctx.pos)
    vis = cache.infer(ctx.positions)
    vis = vis if isinstance(vis, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(vis, np.float32))
    return vis.to(ctx.device, torch.float32).contiguous()


def nls_weights_batch(ctx: PixelCtx, cache, clamp_floor: float | None = CLAMP_FLOOR) -> np.ndarray:
    ctx = as_pixel_ctx(ctx)
    vis = np.asarray(cache.infer(ctx.positions), dtype=np.float64)
    vis = clamp_visibility(vis, clamp_floor) if clamp_floor and clamp_floor > 0.0 else np.maximum(vis, 0.0)
    return vis * ctx.lum_matrix()


def nls_sample_device(ctx: PixelCtx, cache, key: int, offset: int = 0, clamp_floor=CLAMP_FLOOR,
                      p_first: int = 0, p_total: int | None = None, out=None, select_stream=None):
    """Device-resident NLS: returns (ids int64, pts (P,3) f64, W f64) CUDA tensors.

    Pixels of ctx are rows p_first.. of a p_total-pixel frame (screen-tile shard).
    With ``select_stream`` the encoder + MLP run on the current stream and the
    reservoir selection on ``select_stream`` (it can then overlap whatever the
    caller launches next, e.g. the next frame's train step); the outputs are
    ready when ``cache.select_done`` (a CUDA event) completes."""
    ctx = as_pixel_ctx(ctx)
    import torch
    p = ctx.n
    k = ctx.dscene.n_lights
    total = p if p_total is None else p_total
    if out is None:
        out = (torch.empty(p, dtype=torch.int64, device=ctx.device),
               torch.empty((p, 3), dtype=torch.float64, device=ctx.device),
               torch.empty(p, dtype=torch.float64, device=ctx.device))
    ids, pts, big_w = out
    floor = float(clamp_floor) if clamp_floor and clamp_floor > 0.0 else 0.0
    lum = ctx.lum_device()
    lum64 = int(lum.dtype == torch.float64)
    if _is_native(cache) and cache.output_dim != k:
        raise ValueError(f"cache has {cache.output_dim} outputs, scene has {k} lights")
    if _fused(cache):
        ws = cache.query_workspace(p)
        mask = _lib.ptr(ctx.mask_device("lum"))
        if select_stream is None:
            _lib.call("nvc_nls_sample", cache.model, ctx.dscene.struct, ctx.pos.data_ptr(), lum.data_ptr(), lum64,
                      mask, lum.shape[1], p, p_first, total, key, offset, floor, ids.data_ptr(), pts.data_ptr(),
                      big_w.data_ptr(), _lib.ptr(ws), _lib.stream_ptr())
        else:
            cur = torch.cuda.current_stream()
            _lib.call("nvc_query_front", cache.model, ctx.pos.data_ptr(), p, _lib.ptr(ws), _lib.stream_ptr())
            front = torch.cuda.Event()
            front.record(cur)
            select_stream.wait_event(front)
            _lib.call("nvc_nls_select", cache.model, ctx.dscene.struct, lum.data_ptr(), lum64, mask, lum.shape[1], p,
                      p_first, total, key, offset, floor, ids.data_ptr(), pts.data_ptr(), big_w.data_ptr(),
                      _lib.ptr(ws), select_stream.cuda_stream)
            done = torch.cuda.Event()
            done.record(select_stream)
            cache.select_done = done
            # the selection reads / writes these on select_stream: keep the caching
            # allocator from recycling them before it finishes, even if the caller
            # drops the context or the outputs first
            for t in (lum, ctx.mask_device("lum"), ws, ids, pts, big_w):
                t.record_stream(select_stream)
    else:
        vis = _visibility_device(ctx, cache)
        _lib.call("nvc_nls_from_vis", ctx.dscene.struct, vis.data_ptr(), lum.data_ptr(), lum64, lum.shape[1], p,
                  k, p_first, total, key, offset, floor, ids.data_ptr(), pts.data_ptr(), big_w.data_ptr(),
                  _lib.stream_ptr())
    return ids, pts, big_w


def nls_sample_batch(ctx: PixelCtx, cache, rng, clamp_floor: float | None = CLAMP_FLOOR):
    """Exhaustive-stream WRS over all lights: (light ids, emitter points, W = w_sum/w_sel)."""
    ctx = as_pixel_ctx(ctx)
    key, off = rngmod.position(rng)
    ids, pts, big_w = nls_sample_device(ctx, cache, key, off, clamp_floor)
    k = ctx.dscene.n_lights
    rngmod.advance(rng, ctx.n * k + 2 * ctx.n)
    return ids.cpu().numpy(), pts.cpu().numpy(), big_w.cpu().numpy()


def nls_sample(sp: ShadingPoint, cache, scene, rng, clamp_floor: float | None = CLAMP_FLOOR):
    ids, pts, ws = nls_sample_batch(_ctx_for(sp, scene), cache, rng, clamp_floor)
    return int(ids[0]), pts[0], float(ws[0])


def neural_di_device(ctx: PixelCtx, cache, out=None):
    ctx = as_pixel_ctx(ctx)
    import torch
    p = ctx.n
    if out is None:
        out = torch.empty((p, 3), dtype=torch.float64, device=ctx.device)
    if _fused(cache):
        fac = ctx.factor_device()
        _lib.call("nvc_neural_di", cache.model, ctx.dscene.struct, ctx.pos.data_ptr(), ctx.alb.data_ptr(),
                  fac.data_ptr(), int(fac.dtype == torch.float64), _lib.ptr(ctx.mask_device("factor")),
                  fac.shape[1], p, out.data_ptr(), _lib.ptr(cache.query_workspace(p)), _lib.stream_ptr())
        return out
    # unshadowed_rgb (sampling.py:157-160) on the device: (v * f) @ L_e * albedo / pi
    vis = _visibility_device(ctx, cache).to(torch.float64)
    f = ctx.factor_device().to(torch.float64).T
    out.copy_(((vis * f) @ ctx.dscene.lt_radiance) * ctx.alb / np.pi)
    return out


def neural_di_batch(ctx: PixelCtx, cache) -> np.ndarray:
    """Biased shading: predicted visibility times analytic radiance (sampling.py:215-218)."""
    return neural_di_device(ctx, cache).cpu().numpy()


def neural_di_shade(sp: ShadingPoint, cache, scene) -> np.ndarray:
    return neural_di_batch(_ctx_for(sp, scene), cache)[0]


# ---------------------------------------------------------------------------
# clustered NVC: two-step sampling (sampling.py:302-359)
# ---------------------------------------------------------------------------

CLUSTER_TABLE_MAX_BYTES = 32 << 30   # the cluster-ordered copy doubles the factor table's footprint


def _cluster_factor_table(ctx, fac, clusters, c_mem):
    """(p, members) f64 copy of the light-major factor table, columns in the
    ClusterSet's member order (nvc_cluster_factor_table); cached on the context
    per ClusterSet.  None when it would not fit CLUSTER_TABLE_MAX_BYTES."""
    import torch
    n = int(c_mem.numel())
    if os.environ.get("NVC_CLUSTER_LIGHT_MAJOR") or ctx.n * n * 8 > CLUSTER_TABLE_MAX_BYTES:
        return None
    cached = ctx.__dict__.setdefault("_nvc_cluster_ct", {})
    key = id(clusters)
    if key not in cached or cached[key][0] is not clusters:
        out = torch.empty((ctx.n, n), dtype=torch.float64, device=ctx.device)
        _lib.call("nvc_cluster_factor_table", fac.data_ptr(), ctx.n, n, c_mem.data_ptr(), out.data_ptr(),
                  _lib.stream_ptr())
        cached[key] = (clusters, out)
    return cached[key][1]


def clustered_sample_device(ctx: PixelCtx, cache, clusters, key: int, offset: int = 0,
                            clamp_floor=CLAMP_FLOOR):
    """Device tensors (ids, pts, W) and the number of draws consumed."""
    ctx = as_pixel_ctx(ctx)
    import torch
    from .training import _cluster_tables
    m = clusters.m
    vis = _visibility_device(ctx, cache)
    if vis.shape[1] < m:
        raise ValueError(f"cache has {vis.shape[1]} outputs, the ClusterSet {m} clusters")
    p = ctx.n
    ids = torch.empty(p, dtype=torch.int64, device=ctx.device)
    pts = torch.empty((p, 3), dtype=torch.float64, device=ctx.device)
    big_w = torch.empty(p, dtype=torch.float64, device=ctx.device)
    lib = _lib.load()
    ws = torch.empty(lib.nvc_clustered_workspace_bytes(p, m), dtype=torch.uint8, device=ctx.device)
    c_off, c_mem = _cluster_tables(clusters, ctx.device)
    floor = float(clamp_floor) if clamp_floor and clamp_floor > 0.0 else 0.0
    # an f64 per-camera factor table replaces the per-(pixel, member) FP64 factor
    # evaluation with one load (same values); like the reference (render.py:138,
    # FACTOR_CACHE_LIMIT) it is built only up to 64 M (pixel, light) pairs
    k = ctx.dscene.n_lights
    use_table = ctx.table_dtype == np.float64 and (ctx._factor is not None or p * k <= FACTOR_CACHE_LIMIT)
    fac = ctx.factor_device() if use_table else None
    # with a table: read it as the cluster-ordered pixel-major copy (a pixel's
    # candidate members contiguous; built once per (camera, ClusterSet)) -- the
    # light-major rows are gathered 8 B per (pixel, member) from scattered rows
    ct = _cluster_factor_table(ctx, fac, clusters, c_mem) if use_table else None
    if ct is not None:
        _lib.call("nvc_clustered_select_ct", ctx.dscene.struct, vis.data_ptr(), vis.shape[1], ctx.pos.data_ptr(),
                  ctx.nrm.data_ptr(), ctx.alb.data_ptr(), ct.data_ptr(), ct.shape[1], p, m, c_off.data_ptr(),
                  c_mem.data_ptr(), key, offset, floor, ids.data_ptr(), pts.data_ptr(), big_w.data_ptr(),
                  ws.data_ptr(), _lib.stream_ptr())
    else:
        _lib.call("nvc_clustered_select", ctx.dscene.struct, vis.data_ptr(), vis.shape[1], ctx.pos.data_ptr(),
                  ctx.nrm.data_ptr(), ctx.alb.data_ptr(), _lib.ptr(fac), p, m, c_off.data_ptr(), c_mem.data_ptr(),
                  key, offset, floor, ids.data_ptr(), pts.data_ptr(), big_w.data_ptr(), ws.data_ptr(),
                  _lib.stream_ptr())
    lp = ws.view(torch.int64)[lib.nvc_clustered_state_offset(p, m) // 8]
    return ids, pts, big_w, lp + 2 * p - offset


def clustered_sample_batch(ctx: PixelCtx, cache, clusters, rng, clamp_floor: float | None = CLAMP_FLOOR):
    """Cluster WRS on predicted cluster visibility, then streaming RIS over the
    chosen cluster's members; W_total = m * w_sum2 / (m_y * phat(x)).
    Returns (light ids, emitter points, W_total)."""
    key, off = rngmod.position(rng)
    ids, pts, big_w, used = clustered_sample_device(ctx, cache, clusters, key, off, clamp_floor)
    rngmod.advance(rng, int(used.item()))
    return ids.cpu().numpy(), pts.cpu().numpy(), big_w.cpu().numpy()


def clustered_sample(sp: ShadingPoint, cache, clusters, scene, rng, clamp_floor: float | None = CLAMP_FLOOR):
    ids, pts, ws = clustered_sample_batch(_ctx_for(sp, scene), cache, clusters, rng, clamp_floor)
    return int(ids[0]), pts[0], float(ws[0])
