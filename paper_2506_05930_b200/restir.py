"""RIS and screen-space ReSTIR baselines on the GPU (reference sampling.py:365-637).

The reference uses these as the paper's comparison modes (``render_frame``
modes "ris", "restir", "cnvc-restir"; render.py:311-360).  Same functions,
same arguments, same numpy stream consumption; the reservoir grids live on
the device (``ReservoirGrid``: struct of arrays, numpy views on demand):

* ``ris_initial_batch``  -- integers(0, K, (p, M)) candidates (Lemire's bounded
  draw on 32-bit halves, rejections and the kept half exact), luminance target
  weights, streaming WRS, light points (``nvc_ris_initial``);
* ``restir_temporal_batch`` -- history-clamped merge with the previous frame's
  reservoirs, one draw per pixel (``nvc_restir_temporal``);
* ``restir_spatial_batch`` -- ``neighbors`` rounds of random in-radius
  neighbour merges with the normal / depth tests, three draw blocks per round
  (``nvc_restir_spatial``);
* ``cnvc_initial_batch`` -- clustered samples packaged as M = 1 reservoirs.

Candidate ids, WRS choices and draw positions are bit-exact; target weights
use the device FP64 factor table (the numba factor kernel restated, ~1e-12),
so W values agree to ~1e-10 and a merge decision could only differ where
u * w_sum lands within that of w_n.  The spatial offsets go through
rint(r cos / sin(angle)) with CUDA's FP64 cos / sin (<= 2 ulp from libm),
which changes an offset only when r cos(angle) is within ~1e-15 of a
half-integer.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from . import rng as rngmod
from .sampling import CLAMP_FLOOR, Reservoir, ShadingPoint, _ctx_for, as_pixel_ctx

RESTIR_CANDIDATES = 8
RESTIR_RADIUS = 32
RESTIR_NEIGHBORS = 4
RESTIR_TEMPORAL_CLAMP = 20.0
_FIELDS = ("y", "point", "w_y", "w_sum", "M", "W", "valid")


class ReservoirGrid:
    """One reservoir per pixel, struct of arrays on the device (sampling.py:369-402).
    Attribute reads (y, point, w_y, w_sum, M, W, valid) return host numpy copies."""

    def __init__(self, n: int, device=None):
        torch = _lib.require_cuda()
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.d = {"y": torch.full((n,), -1, dtype=torch.int64, device=dev),
                  "point": torch.zeros((n, 3), dtype=torch.float64, device=dev),
                  **{k: torch.zeros(n, dtype=torch.float64, device=dev) for k in ("w_y", "w_sum", "M", "W")},
                  "valid": torch.zeros(n, dtype=torch.uint8, device=dev)}
        self.device = dev

    @classmethod
    def of(cls, grid, device):
        """This class for `grid` (a reference ReservoirGrid is uploaded)."""
        if isinstance(grid, ReservoirGrid):
            return grid
        import torch
        out = cls(grid.y.shape[0], device)
        for k in _FIELDS:
            v = np.asarray(getattr(grid, k))
            out.d[k].copy_(torch.from_numpy(np.ascontiguousarray(v.astype(np.uint8) if k == "valid" else v)))
        return out

    def __getattr__(self, name):
        if name in _FIELDS:
            v = self.d[name].cpu().numpy()
            return v.astype(bool) if name == "valid" else v
        raise AttributeError(name)

    @property
    def n(self) -> int:
        return self.d["y"].shape[0]

    def invalidate(self) -> None:
        self.d["valid"].zero_()

    def struct(self) -> _lib.NvcRGrid:
        g = _lib.NvcRGrid()
        for k in _FIELDS:
            setattr(g, k, self.d[k].data_ptr())
        return g

    def row(self, i: int) -> Reservoir:
        return Reservoir(y=int(self.y[i]), point=self.point[i].copy(), w_y=float(self.w_y[i]),
                         w_sum=float(self.w_sum[i]), M=float(self.M[i]), W=float(self.W[i]))

    def set_row(self, i: int, r: Reservoir, valid: bool = True) -> None:
        import torch
        self.d["y"][i] = int(r.y)
        if r.point is not None:
            self.d["point"][i] = torch.as_tensor(np.asarray(r.point, np.float64))
        for k in ("w_y", "w_sum", "M", "W"):
            self.d[k][i] = float(getattr(r, k))
        self.d["valid"][i] = int(valid)


def _factor(ctx):
    import torch
    f = ctx.factor_device()
    return f if f.dtype == torch.float64 else f.to(torch.float64)


def ris_initial_batch(ctx, rng, m_candidates: int = RESTIR_CANDIDATES) -> ReservoirGrid:
    """Streaming RIS over uniformly drawn light candidates (sampling.py:405-432):
    W = w_sum / (M * phat(y))."""
    import torch
    ctx = as_pixel_ctx(ctx)
    p, k = ctx.n, ctx.dscene.n_lights
    key, off = rngmod.position(rng)
    kept = -1
    if not isinstance(rng, rngmod.Stream) and rng.bit_generator.state.get("has_uint32"):
        kept = int(rng.bit_generator.state["uinteger"])
    lum = ctx.lum_device()
    out = ReservoirGrid(p, ctx.device)
    ws = torch.empty(int(_lib.load().nvc_ris_workspace_bytes(p, m_candidates, k)), dtype=torch.uint8,
                     device=ctx.device)
    state = torch.empty(2, dtype=torch.int64, device=ctx.device)
    _lib.call("nvc_ris_initial", ctx.dscene.struct, lum.data_ptr(), int(lum.dtype == torch.float64), lum.shape[1], p,
              m_candidates, key, off, kept, out.struct(), ws.data_ptr(), state.data_ptr(), _lib.stream_ptr())
    first, kept_after = (int(x) for x in state.cpu())
    if isinstance(rng, rngmod.Stream):
        rng.offset = first + p * m_candidates + 2 * p
    else:
        rngmod.set_position(rng, first + p * m_candidates + 2 * p)
        rngmod.set_kept32(rng, None if kept_after < 0 else kept_after)
    return out


def ris_initial_candidates(sp: ShadingPoint, scene, rng, m_candidates: int = RESTIR_CANDIDATES) -> Reservoir:
    if m_candidates < 1:
        raise ValueError("need at least one candidate")
    return ris_initial_batch(_ctx_for(sp, scene), rng, m_candidates).row(0)


def cnvc_initial_batch(ctx, cache, clusters, rng, clamp_floor: float | None = CLAMP_FLOOR) -> ReservoirGrid:
    """Clustered samples as ReSTIR-compatible reservoirs, M = 1 (sampling.py:441-461)."""
    import torch
    from .sampling import clustered_sample_device
    ctx = as_pixel_ctx(ctx)
    key, off = rngmod.position(rng)
    ids, pts, big_w, used = clustered_sample_device(ctx, cache, clusters, key, off, clamp_floor)
    rngmod.advance(rng, int(used.item()))
    out = ReservoirGrid(ctx.n, ctx.device)
    w_y = out.d["w_y"]
    f = _factor(ctx)
    _lib.call("nvc_phat_ids", ctx.dscene.struct, f.data_ptr(), f.shape[1], ctx.alb.data_ptr(), ids.data_ptr(),
              ctx.n, w_y.data_ptr(), _lib.stream_ptr())
    out.d["y"].copy_(ids)
    out.d["point"].copy_(pts)
    out.d["M"].fill_(1.0)
    out.d["W"].copy_(torch.where(w_y > 0, big_w, torch.zeros_like(big_w)))
    out.d["w_sum"].copy_(w_y * out.d["W"])
    out.d["valid"].fill_(1)
    return out


def cnvc_initial_candidates(sp: ShadingPoint, cache, clusters, scene, rng,
                            clamp_floor: float | None = CLAMP_FLOOR) -> Reservoir:
    return cnvc_initial_batch(_ctx_for(sp, scene), cache, clusters, rng, clamp_floor).row(0)


def restir_temporal_batch(cur, prev, ctx, rng, clamp: float = RESTIR_TEMPORAL_CLAMP,
                          clamp_mode: str = "m") -> ReservoirGrid:
    """Merge each pixel's previous reservoir into the current one (sampling.py:487-526)."""
    if clamp_mode not in ("m", "contribution"):
        raise ValueError(f"unknown clamp mode {clamp_mode!r}")
    ctx = as_pixel_ctx(ctx)
    cur, prev = ReservoirGrid.of(cur, ctx.device), ReservoirGrid.of(prev, ctx.device)
    out = ReservoirGrid(cur.n, ctx.device)
    key, off = rngmod.position(rng)
    f = _factor(ctx)
    _lib.call("nvc_restir_temporal", ctx.dscene.struct, f.data_ptr(), f.shape[1], ctx.alb.data_ptr(), cur.n,
              cur.struct(), prev.struct(), key, off, float(clamp), int(clamp_mode == "contribution"), out.struct(),
              _lib.stream_ptr())
    rngmod.advance(rng, cur.n)
    return out


def restir_temporal(current: Reservoir, previous, sp: ShadingPoint, scene, rng,
                    clamp: float = RESTIR_TEMPORAL_CLAMP, clamp_mode: str = "m") -> Reservoir:
    """Scalar temporal merge; previous=None means first frame / disocclusion."""
    if previous is None:
        return current
    cur, prev = ReservoirGrid(1), ReservoirGrid(1)
    cur.set_row(0, current)
    prev.set_row(0, previous)
    return restir_temporal_batch(cur, prev, _ctx_for(sp, scene), rng, clamp, clamp_mode).row(0)


def restir_spatial_batch(grid, ctx, shape, hit, depth, normals, rng, radius: int = RESTIR_RADIUS,
                         neighbors: int = RESTIR_NEIGHBORS) -> ReservoirGrid:
    """Merge random in-radius neighbour reservoirs (sampling.py:541-595); neighbours
    are rejected when either pixel missed, normals disagree (dot < 0.9) or depths
    differ by more than 10 %."""
    import torch
    ctx = as_pixel_ctx(ctx)
    g = ReservoirGrid.of(grid, ctx.device)
    h, w = shape
    dev = ctx.device
    as_t = (lambda a, dt: a.to(dev, dt).contiguous() if isinstance(a, torch.Tensor)
            else torch.from_numpy(np.ascontiguousarray(a)).to(dev, dt))
    hit_t = as_t(np.asarray(hit).astype(np.uint8) if not isinstance(hit, torch.Tensor) else hit, torch.uint8)
    depth_t = as_t(depth, torch.float64).reshape(-1)
    nrm_t = as_t(normals, torch.float64).reshape(-1, 3)
    out = ReservoirGrid(g.n, dev)
    key, off = rngmod.position(rng)
    f = _factor(ctx)
    _lib.call("nvc_restir_spatial", ctx.dscene.struct, f.data_ptr(), f.shape[1], ctx.alb.data_ptr(),
              nrm_t.data_ptr(), hit_t.data_ptr(), depth_t.data_ptr(), w, h, g.struct(), key, off, int(radius),
              int(neighbors), out.struct(), _lib.stream_ptr())
    rngmod.advance(rng, 3 * neighbors * g.n)
    return out


def restir_spatial(pixel, grid, gbuffer, scene, rng, radius: int = RESTIR_RADIUS,
                   neighbors: int = RESTIR_NEIGHBORS) -> Reservoir:
    """Scalar spatial reuse for one (x, y) pixel against a full grid
    (sampling.py:598-637): the reference's scalar draw order (angle, radius,
    merge uniform per neighbour), target weights through the device phat."""
    px, py = pixel
    h, w = gbuffer.shape
    i = py * w + px
    pos = np.asarray(gbuffer.position).reshape(-1, 3)
    nrm = np.asarray(gbuffer.normal).reshape(-1, 3)
    alb = np.asarray(gbuffer.albedo).reshape(-1, 3)
    hit = np.asarray(gbuffer.hit).reshape(-1)
    depth = np.asarray(gbuffer.depth).reshape(-1)
    ctx = _ctx_for(ShadingPoint(pos[i], nrm[i], alb[i]), scene)
    ys, Ws, Ms, valid, pts = grid.y, grid.W, grid.M, grid.valid, grid.point
    phat = lambda y: float(ctx.phat_ids(np.array([y]))[0])   # noqa: E731
    acc = Reservoir(y=int(ys[i]), point=pts[i].copy(), W=float(Ws[i]), M=float(Ms[i]))
    acc_wsum = phat(acc.y) * acc.W * acc.M
    acc_m = acc.M
    for _ in range(neighbors):
        ang = rng.random() * 2.0 * np.pi
        rad = radius * np.sqrt(rng.random())
        dx, dy = int(np.rint(rad * np.cos(ang))), int(np.rint(rad * np.sin(ang)))
        nx, ny = px + dx, py + dy
        u = rng.random()
        if (dx == 0 and dy == 0) or not (0 <= nx < w and 0 <= ny < h):
            continue
        j = ny * w + nx
        if not (valid[j] and hit[i] and hit[j]) or nrm[i] @ nrm[j] < 0.9:
            continue
        ratio = depth[j] / max(depth[i], 1e-12)
        if not (0.9 <= ratio <= 1.1):
            continue
        w_n = phat(int(ys[j])) * Ws[j] * Ms[j]
        w_sum = acc_wsum + w_n
        if w_n > 0 and u * w_sum < w_n:
            acc.y, acc.point = int(ys[j]), pts[j].copy()
        acc_wsum = w_sum
        acc_m += Ms[j]
    ph = phat(acc.y)
    if acc_wsum > 0 and ph > 0 and acc_m > 0:
        return Reservoir(y=acc.y, point=acc.point, w_y=ph, w_sum=acc_wsum, M=acc_m, W=acc_wsum / (acc_m * ph))
    return Reservoir(M=acc_m, w_sum=acc_wsum)


__all__ = ["ReservoirGrid", "ris_initial_batch", "ris_initial_candidates", "cnvc_initial_batch",
           "cnvc_initial_candidates", "restir_temporal_batch", "restir_temporal", "restir_spatial_batch",
           "restir_spatial", "RESTIR_CANDIDATES", "RESTIR_RADIUS", "RESTIR_NEIGHBORS", "RESTIR_TEMPORAL_CLAMP"]
