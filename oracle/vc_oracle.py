"""CPU oracle for the neural-visibility-cache hot path -- TEST INFRASTRUCTURE.

This module is the parity checker, never the product: only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  It restates the reference
``viscache`` 0.1.0 algorithm (``/root/reference/pkg/src/viscache``) in numpy
plus a plain-C geometry core (``oracle/geom.c``), with every function citing
the reference file:line it follows.  Parity is PINNED: ``tests/test_oracle.py``
checks each function against the golden vectors that
``tests/golden/make_golden.py`` produced by running the reference itself.

Third-party arithmetic the reference delegates (numpy 2.3.x, installed here):
numpy ``Philox`` 4x64-10 (restated below, pinned against numpy's own
``Generator``), ``np.einsum`` blend order (restated as a sequential FP32
accumulate, pinned by golden features), ``np.cumsum`` (sequential FP64),
``np.add.at`` (sequential scatter), OpenBLAS sgemm (used as-is: MLP matmuls are
compared within the tolerance the reference's own tests use, 1e-6).
"""

from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
M64 = (1 << 64) - 1

# ---------------------------------------------------------------------------
# RNG: rng.py:30-56 (stream_key) + numpy Philox4x64-10 (random access)
# ---------------------------------------------------------------------------

PURPOSE = {"primary": "primary", "world": "world-samples", "screen": "screen-samples",
           "targets": "targets", "select": "light-select", "init": "init-params"}


def _splitmix64(x: int) -> int:          # rng.py:30-35
    x = (x + 0x9E3779B97F4A7C15) & M64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & M64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & M64
    return x ^ (x >> 31)


def _fnv1a64(s: str) -> int:             # rng.py:38-42
    h = 0xCBF29CE484222325
    for byte in s.encode("utf-8"):
        h = ((h ^ byte) * 0x100000001B3) & M64
    return h


def stream_key(*parts) -> int:           # rng.py:45-51
    h = 0x8000000000000001
    for p in parts:
        h = _splitmix64(h ^ (_fnv1a64(p) if isinstance(p, str) else (p & M64)))
    return h


_PM0, _PM1 = np.uint64(0xD2E7470EE14C6C93), np.uint64(0xCA5A826395121157)
_PW0, _PW1 = np.uint64(0x9E3779B97F4A7C15), np.uint64(0xBB67AE8584CAA73B)
_LO32 = np.uint64(0xFFFFFFFF)
_S32 = np.uint64(32)


def _mulhilo(a: np.uint64, b: np.ndarray):
    """64x64 -> 128 product split into 32-bit limbs (numpy uint64 wraps)."""
    al, ah = a & _LO32, a >> _S32
    bl, bh = b & _LO32, b >> _S32
    p0, p1, p2, p3 = al * bl, al * bh, ah * bl, ah * bh
    mid = (p0 >> _S32) + (p1 & _LO32) + (p2 & _LO32)
    hi = p3 + (p1 >> _S32) + (p2 >> _S32) + (mid >> _S32)
    return hi, a * b


def philox_blocks(key: int, counters: np.ndarray) -> np.ndarray:
    """Philox4x64-10 of counter [c, 0, 0, 0], key [key, 0]; returns (n, 4)."""
    c0 = np.asarray(counters, dtype=np.uint64)
    c1 = np.zeros_like(c0)
    c2 = np.zeros_like(c0)
    c3 = np.zeros_like(c0)
    k0, k1 = np.uint64(key & M64), np.uint64(0)
    with np.errstate(over="ignore"):
        for r in range(10):
            if r:
                k0 = k0 + _PW0
                k1 = k1 + _PW1
            hi0, lo0 = _mulhilo(_PM0, c0)
            hi1, lo1 = _mulhilo(_PM1, c2)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
    return np.stack([c0, c1, c2, c3], axis=-1)


def raw_at(key: int, idx) -> np.ndarray:
    """uint64 draw number ``idx`` of the stream (draw n = lane n%4 of block n//4+1)."""
    idx = np.asarray(idx, dtype=np.int64)
    flat = idx.reshape(-1)
    blocks = philox_blocks(key, (flat // 4 + 1).astype(np.uint64))
    return blocks[np.arange(flat.size), flat % 4].reshape(idx.shape)


def uniform_at(key: int, idx) -> np.ndarray:
    """Generator.random() value of draw ``idx``: (x >> 11) * 2^-53."""
    return (raw_at(key, idx) >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


class Stream:
    """Sequential view of a counter-based stream (what rng.stream returns)."""

    def __init__(self, *parts, key: int | None = None, offset: int = 0):
        self.key = stream_key(*parts) if key is None else key
        self.offset = offset

    def random(self, shape) -> np.ndarray:
        n = int(np.prod(shape))
        out = uniform_at(self.key, np.arange(self.offset, self.offset + n)).reshape(shape)
        self.offset += n
        return out

    def uniform(self, lo, hi, shape) -> np.ndarray:   # numpy: lo + (hi - lo) * u
        u = self.random(shape)
        return np.asarray(lo) + (np.asarray(hi) - np.asarray(lo)) * u


# ---------------------------------------------------------------------------
# Hash-grid encoder: hashgrid.py:22-151
# ---------------------------------------------------------------------------

PRIMES = (1, 2654435761, 805459861)      # hashgrid.py:20


class Grid:
    """HashGridConfig restated (hashgrid.py:32-65)."""

    def __init__(self, levels=10, base_resolution=16, per_level_scale=(512.0 / 16.0) ** (1.0 / 9.0),
                 features_per_level=4, table_size=1 << 14, aabb_min=(0, 0, 0), aabb_max=(1, 1, 1)):
        self.levels, self.base, self.scale = levels, base_resolution, per_level_scale
        self.F, self.T = features_per_level, table_size
        self.lo = np.asarray(aabb_min, dtype=np.float64)
        self.hi = np.asarray(aabb_max, dtype=np.float64)

    def res(self, l: int) -> int:                  # hashgrid.py:60-61
        return int(np.floor(self.base * self.scale ** l))

    def dense(self, l: int) -> bool:               # hashgrid.py:63-65
        n = self.res(l) + 1
        return n * n * n <= self.T


def normalize(g: Grid, pos: np.ndarray) -> np.ndarray:    # hashgrid.py:94-97
    span = np.maximum(g.hi - g.lo, 1e-12)
    return np.clip((np.asarray(pos, dtype=np.float64) - g.lo) / span, 0.0, 1.0)


def level_lookup(g: Grid, l: int, q: np.ndarray):         # hashgrid.py:100-114, 82-87
    n = g.res(l)
    x = q * n
    c0 = np.minimum(x.astype(np.int64), n - 1)
    f = x - c0
    idx = np.empty((q.shape[0], 8), dtype=np.int64)
    w = np.empty((q.shape[0], 8), dtype=np.float64)
    for c in range(8):                        # corner c = 4*bx + 2*by + bz
        b = ((c >> 2) & 1, (c >> 1) & 1, c & 1)
        cc = [c0[:, a] + b[a] for a in range(3)]
        wa = [f[:, a] if b[a] else 1.0 - f[:, a] for a in range(3)]
        w[:, c] = (wa[0] * wa[1]) * wa[2]
        if g.dense(l):
            m = n + 1
            idx[:, c] = cc[0] + m * (cc[1] + m * cc[2])
        else:
            h = (cc[0] * PRIMES[0] + cc[1] * PRIMES[1] + cc[2] * PRIMES[2])
            idx[:, c] = h & (g.T - 1)
    return idx, w


def encode(g: Grid, table: np.ndarray, pos: np.ndarray):  # hashgrid.py:117-131
    """Features (B, L*F) in the table dtype; blend = sequential acc + w_c*f_c."""
    q = normalize(g, pos)
    out = np.empty((q.shape[0], g.levels * g.F), dtype=table.dtype)
    ctx = []
    for l in range(g.levels):
        idx, w = level_lookup(g, l, q)
        wt = w.astype(table.dtype)
        acc = np.zeros((q.shape[0], g.F), dtype=table.dtype)
        for c in range(8):
            acc = acc + wt[:, c, None] * table[l][idx[:, c]]
        out[:, l * g.F:(l + 1) * g.F] = acc
        ctx.append((idx, w))
    return out, ctx


def grid_grad(g: Grid, ctx, up: np.ndarray, dtype=np.float32) -> np.ndarray:   # hashgrid.py:140-151
    grad = np.zeros((g.levels, g.T, g.F), dtype=dtype)
    for l, (idx, w) in enumerate(ctx):
        contrib = (w[:, :, None] * up[:, None, l * g.F:(l + 1) * g.F]).astype(dtype)
        np.add.at(grad[l], idx.reshape(-1), contrib.reshape(-1, g.F))
    return grad


# ---------------------------------------------------------------------------
# MLP + Adam: mlp.py:63-218
# ---------------------------------------------------------------------------

def lr_at(step: int, lr_start=0.05, lr_end=0.001, warm=200) -> float:   # mlp.py:76-81
    return lr_start + (lr_end - lr_start) * (min(step, warm) / warm)


def he_weights(dims, stream_gen, dtype=np.float32):                   # mlp.py:84-90
    ws, bs = [], []
    for fo, fi in zip(dims[1:], dims[:-1]):
        ws.append(stream_gen.normal(0.0, math.sqrt(2.0 / fi), (fo, fi)).astype(dtype))
        bs.append(np.zeros(fo, dtype=dtype))
    return ws, bs


def mlp_forward(ws, bs, x, alpha=0.01):                               # mlp.py:110-140
    a = np.asarray(x, dtype=ws[0].dtype)
    acts, zs = [a], []
    for i, (w, b) in enumerate(zip(ws, bs)):
        z = a @ w.T + b
        zs.append(z)
        if i < len(ws) - 1:
            a = np.where(z >= 0, z, alpha * z)
        else:
            a = np.empty_like(z)
            p = z >= 0
            a[p] = 1.0 / (1.0 + np.exp(-z[p]))
            e = np.exp(z[~p])
            a[~p] = e / (1.0 + e)
        acts.append(a)
    return np.clip(acts[-1], 1e-6, 1.0 - 1e-6), zs, acts


def l2_loss(out, t, mask=None) -> float:                               # mlp.py:143-149
    d = out - t
    if mask is not None:
        d = d * mask
    return float(np.mean(np.sum(d * d, axis=1) / out.shape[1]))


def mlp_backward(ws, zs, acts, t, mask=None, alpha=0.01, b_scale=None):   # mlp.py:152-183
    out = acts[-1]
    b, k = out.shape
    d_out = 2.0 * (out - t) / ((b if b_scale is None else b_scale) * k)
    if mask is not None:
        d_out = d_out * mask
    dz = d_out * out * (1.0 - out)
    gw, gb = [None] * len(ws), [None] * len(ws)
    d_in = None
    for i in range(len(ws) - 1, -1, -1):
        gw[i] = dz.T @ acts[i]
        gb[i] = dz.sum(axis=0)
        da = dz @ ws[i]
        if i > 0:
            dz = da * np.where(zs[i - 1] >= 0, 1.0, alpha).astype(da.dtype)
        else:
            d_in = da
    return gw, gb, d_in


class Adam:                                                           # mlp.py:186-218
    def __init__(self, n, dtype=np.float32):
        self.m = np.zeros(n, dtype)
        self.v = np.zeros(n, dtype)
        self.t = 0

    def step(self, p, g, lr):
        self.t += 1
        b1c, b2c = 1.0 - 0.9 ** self.t, 1.0 - 0.999 ** self.t
        self.m *= 0.9
        self.m += (1.0 - 0.9) * g
        self.v *= 0.999
        self.v += (1.0 - 0.999) * g * g
        p -= lr * (self.m / b1c) / (np.sqrt(self.v / b2c) + 1e-8)


class Cache:
    """VisibilityCache restated (cache.py:25-73) for arbitrary hidden dims.

    Init follows cache.py:41-43: one (seed, "init-params") stream, table first
    (U(+-1e-4), hashgrid.py:75-79), then He weights layer by layer."""

    def __init__(self, grid: Grid, k: int, hidden=(32, 32), seed=0, dtype=np.float32):
        self.grid, self.k = grid, k
        gen = np.random.Generator(np.random.Philox(key=stream_key(seed, "init-params")))
        self.table = gen.uniform(-1e-4, 1e-4, (grid.levels, grid.T, grid.F)).astype(dtype)
        self.dims = [grid.levels * grid.F, *hidden, k]
        self.ws, self.bs = he_weights(self.dims, gen, dtype)
        self.adam = Adam(self.param_count, dtype)
        self.step = 0

    @property
    def param_count(self) -> int:
        return self.table.size + sum(w.size + b.size for w, b in zip(self.ws, self.bs))

    def flat(self) -> np.ndarray:
        parts = [self.table.reshape(-1)]
        for w, b in zip(self.ws, self.bs):
            parts += [w.reshape(-1), b]
        return np.concatenate(parts)

    def unflat(self, v: np.ndarray) -> None:
        o = self.table.size
        self.table[...] = v[:o].reshape(self.table.shape)
        for w, b in zip(self.ws, self.bs):
            w[...] = v[o:o + w.size].reshape(w.shape)
            o += w.size
            b[...] = v[o:o + b.size]
            o += b.size

    def infer(self, pos):
        feats, _ = encode(self.grid, self.table, pos)
        return mlp_forward(self.ws, self.bs, feats)[0]

    def grads(self, pos, tgt, b_scale=None, mask=None):
        feats, ctx = encode(self.grid, self.table, pos)
        out, zs, acts = mlp_forward(self.ws, self.bs, feats)
        loss = l2_loss(out, tgt, mask)
        gw, gb, d_in = mlp_backward(self.ws, zs, acts, tgt, mask=mask, b_scale=b_scale)
        gg = grid_grad(self.grid, ctx, d_in, self.table.dtype)
        parts = [gg.reshape(-1)]
        for w, b in zip(gw, gb):
            parts += [w.reshape(-1), b]
        return loss, np.concatenate(parts)

    def train_step(self, pos, tgt, mask=None) -> float:
        loss, g = self.grads(pos, tgt, mask=mask)
        p = self.flat()
        self.adam.step(p, g, lr_at(self.step))
        self.unflat(p)
        self.step += 1
        return loss


# ---------------------------------------------------------------------------
# Geometry (C core) + scene helpers: geometry.py, scene.py, render.py
# ---------------------------------------------------------------------------

_LIB = None


def lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(HERE, "build", "liboracle_geom.so")
        if not os.path.exists(path):
            build()
        _LIB = ctypes.CDLL(path)
    return _LIB


def build() -> str:
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    out = os.path.join(HERE, "build", "liboracle_geom.so")
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC",
                           "-shared", "-o", out, os.path.join(HERE, "geom.c"), "-lm"])
    return out


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


class Bvh:
    """Median-split BVH restated from geometry.py:97-158 (leaf <= 4, longest
    centroid axis, stable argsort, left = lower half)."""

    def __init__(self, v0, v1, v2):
        v0, v1, v2 = (np.ascontiguousarray(a, dtype=np.float64) for a in (v0, v1, v2))
        n = v0.shape[0]
        if n == 0:
            self.node_min = np.full((1, 3), np.inf)
            self.node_max = np.full((1, 3), -np.inf)
            self.left = np.array([-1], np.int32)
            self.right = np.array([-1], np.int32)
            self.start = np.array([0], np.int32)
            self.count = np.array([0], np.int32)
            self.perm = np.empty(0, np.int64)
            self.v0, self.v1, self.v2 = v0, v1, v2
            return
        cen = (v0 + v1 + v2) / 3.0
        tmin = np.minimum(np.minimum(v0, v1), v2)
        tmax = np.maximum(np.maximum(v0, v1), v2)
        nmin, nmax, left, right, start, count, order = [], [], [], [], [], [], []

        def rec(ids):
            me = len(left)
            nmin.append(tmin[ids].min(axis=0))
            nmax.append(tmax[ids].max(axis=0))
            left.append(-1)
            right.append(-1)
            start.append(0)
            count.append(0)
            if ids.size <= 4:
                start[me] = len(order)
                count[me] = ids.size
                order.extend(ids.tolist())
                return me
            c = cen[ids]
            axis = int(np.argmax(c.max(axis=0) - c.min(axis=0)))
            srt = np.argsort(c[:, axis], kind="stable")
            half = ids.size // 2
            left[me] = rec(ids[srt[:half]])
            right[me] = rec(ids[srt[half:]])
            return me

        rec(np.arange(n))
        self.perm = np.asarray(order, np.int64)
        self.node_min = np.ascontiguousarray(nmin, np.float64)
        self.node_max = np.ascontiguousarray(nmax, np.float64)
        self.left, self.right = np.asarray(left, np.int32), np.asarray(right, np.int32)
        self.start, self.count = np.asarray(start, np.int32), np.asarray(count, np.int32)
        self.v0, self.v1, self.v2 = (np.ascontiguousarray(a[self.perm]) for a in (v0, v1, v2))

    def _args(self):
        return (_p(self.node_min), _p(self.node_max), _p(self.left), _p(self.right),
                _p(self.start), _p(self.count), _p(self.v0), _p(self.v1), _p(self.v2),
                ctypes.c_int64(self.v0.shape[0]))

    def closest(self, o, d, t_min, t_max):
        """(t, original tri index or -1) -- geometry.py:191-207."""
        n = o.shape[0]
        o, d = np.ascontiguousarray(o, np.float64), np.ascontiguousarray(d, np.float64)
        t_min = np.ascontiguousarray(t_min, np.float64)
        t_max = np.ascontiguousarray(t_max, np.float64)
        t = np.empty(n)
        tri = np.empty(n, np.int64)
        lib().orc_closest_hit_batch(ctypes.c_int64(n), _p(o), _p(d), _p(t_min), _p(t_max),
                                    *self._args(), _p(t), _p(tri))
        hit = tri >= 0
        tri[hit] = self.perm[tri[hit]]
        return t, tri

    def occluded(self, o, d, t_min, t_max):
        n = o.shape[0]
        o, d = np.ascontiguousarray(o, np.float64), np.ascontiguousarray(d, np.float64)
        t_min = np.ascontiguousarray(t_min, np.float64)
        t_max = np.ascontiguousarray(t_max, np.float64)
        out = np.empty(n, np.uint8)
        lib().orc_any_hit_batch(ctypes.c_int64(n), _p(o), _p(d), _p(t_min), _p(t_max),
                                *self._args(), _p(out))
        return out.astype(bool)

    @property
    def diagonal(self) -> float:
        return float(np.linalg.norm(self.node_max[0] - self.node_min[0]))


class SceneArrays:
    """The packed scene the reference's Scene carries (scene.py:158-215)."""

    def __init__(self, v0, v1, v2, tri_material, tri_light, lt_kind, lt_verts, lt_normal,
                 lt_radiance, mat_albedo, cam, lt_area=None):
        self.v0, self.v1, self.v2 = v0, v1, v2
        self.lt_area = None if lt_area is None else np.asarray(lt_area, np.float64)
        self.tri_material, self.tri_light = tri_material, tri_light
        self.lt_kind, self.lt_verts = lt_kind.astype(np.uint8), np.ascontiguousarray(lt_verts)
        self.lt_normal, self.lt_radiance = np.ascontiguousarray(lt_normal), lt_radiance
        self.mat_albedo = mat_albedo
        self.cam = cam                     # (pos3, look3, up3, fov, W, H)
        self.bvh = Bvh(v0, v1, v2)
        pts = [v0, v1, v2, lt_verts.reshape(-1, 3)]
        allp = np.concatenate([p.reshape(-1, 3) for p in pts if p.size])
        self.aabb_min, self.aabb_max = allp.min(axis=0), allp.max(axis=0)

    @property
    def k(self) -> int:
        return self.lt_kind.shape[0]

    @classmethod
    def from_golden(cls, z, prefix):
        g = lambda k: z[prefix + k]  # noqa: E731
        return cls(g("v0"), g("v1"), g("v2"), g("tri_material"), g("tri_light"), g("lt_kind"),
                   g("lt_verts"), g("lt_normal"), g("lt_radiance"), g("mat_albedo"), g("cam"),
                   lt_area=g("lt_area") if prefix + "lt_area" in z else None)

    def light_points(self, ids, u):                                   # scene.py:204-215
        safe = np.maximum(np.asarray(ids), 0)
        verts = self.lt_verts[safe]
        pts = verts[:, 0] + u[:, :1] * (verts[:, 1] - verts[:, 0]) + u[:, 1:2] * (verts[:, 3] - verts[:, 0])
        is_pt = self.lt_kind[safe] == 1
        pts[is_pt] = verts[is_pt, 0]
        return pts

    def camera_rays(self, sx, sy, width=None, height=None):           # scene.py:109-139
        pos, look, up = self.cam[0:3], self.cam[3:6], self.cam[6:9]
        fov = self.cam[9]
        w = int(self.cam[10]) if width is None else width
        h = int(self.cam[11]) if height is None else height
        fwd = look - pos
        fwd = fwd / np.linalg.norm(fwd)
        right = np.cross(fwd, up)
        right /= np.linalg.norm(right)
        tup = np.cross(right, fwd)
        th = np.tan(np.radians(fov) * 0.5)
        nx = (2.0 * sx / w - 1.0) * th * (w / h)
        ny = (1.0 - 2.0 * sy / h) * th
        d = fwd[None, :] + nx[:, None] * right[None, :] + ny[:, None] * tup[None, :]
        d /= np.linalg.norm(d, axis=1, keepdims=True)
        return np.broadcast_to(pos, d.shape).copy(), d

    def trace(self, o, d):                                             # render.py:49-75
        n = o.shape[0]
        t, tri = self.bvh.closest(o, d, np.zeros(n), np.full(n, np.inf))
        hit = tri >= 0
        safe = np.maximum(tri, 0)
        pos = o + t[:, None] * d
        nrm = np.cross(self.v1[safe] - self.v0[safe], self.v2[safe] - self.v0[safe])
        nrm /= np.maximum(np.linalg.norm(nrm, axis=1, keepdims=True), 1e-300)
        facing = np.einsum("pc,pc->p", nrm, d) > 0
        nrm[facing] *= -1.0
        mat = self.tri_material[safe]
        alb = np.where((mat >= 0)[:, None], self.mat_albedo[np.maximum(mat, 0)], 0.0)
        return {"hit": hit, "position": np.where(hit[:, None], pos, 0.0),
                "normal": np.where(hit[:, None], nrm, 0.0),
                "albedo": np.where(hit[:, None], alb, 0.0),
                "light_id": np.where(hit, self.tri_light[safe], -1)}

    def gbuffer(self, width=None, height=None):                        # render.py:103-117
        w = int(self.cam[10]) if width is None else width
        h = int(self.cam[11]) if height is None else height
        jit = Stream("primary").random((h * w, 2))
        ys, xs = np.divmod(np.arange(h * w), w)
        o, d = self.camera_rays(xs + jit[:, 0], ys + jit[:, 1], w, h)
        return self.trace(o, d)

    def visibility(self, x, y):                                         # geometry.py:221-247
        d_ = self.bvh.diagonal
        eps = 1e-4 * (d_ if np.isfinite(d_) and d_ > 0.0 else 1.0)
        d = y - x
        dist = np.linalg.norm(d, axis=1)
        dirs = d / np.maximum(dist, 1e-300)[:, None]
        t_min = np.full(x.shape[0], eps)
        t_max = dist - eps
        degenerate = t_max <= t_min
        t_max = np.maximum(t_max, t_min + 1e-12)
        vis = (~self.bvh.occluded(x, dirs, t_min, t_max)).astype(np.float64)
        vis[degenerate] = 1.0
        return vis

    def factors(self, pos, nrm):                                        # kernels.py:299-316
        pos = np.ascontiguousarray(pos, np.float64)
        nrm = np.ascontiguousarray(nrm, np.float64)
        out = np.empty((pos.shape[0], self.k))
        lib().orc_light_factors(ctypes.c_int64(pos.shape[0]), _p(pos), _p(nrm),
                                ctypes.c_int64(self.k), _p(self.lt_kind), _p(self.lt_verts),
                                _p(self.lt_normal), _p(out))
        return out

    def lum(self, factor, albedo):                                      # sampling.py:134-139
        luma = np.array([0.2126, 0.7152, 0.0722])
        return factor * (albedo @ (luma[:, None] * self.lt_radiance.T) / np.pi)


# ---------------------------------------------------------------------------
# Training data: training.py:44-129
# ---------------------------------------------------------------------------

def world_samples(s: SceneArrays, n: int, st: Stream) -> np.ndarray:      # training.py:44-48
    if n == 0:
        return np.zeros((0, 3))
    return st.uniform(s.aabb_min, s.aabb_max, (n, 3))


def screen_samples(s: SceneArrays, n: int, st: Stream, rounds: int = 8) -> np.ndarray:  # :67-100
    w, h = int(s.cam[10]), int(s.cam[11])
    got, want = [], n
    for _ in range(rounds + 1):
        if want == 0:
            break
        sx = st.random(want) * w
        sy = st.random(want) * h
        o, d = s.camera_rays(sx, sy)
        tr = s.trace(o, d)
        got.append(tr["position"][tr["hit"]])
        want -= int(tr["hit"].sum())
    return np.concatenate(got) if got else np.zeros((0, 3))


def targets(s: SceneArrays, pos: np.ndarray, st: Stream) -> np.ndarray:    # training.py:103-120
    b = pos.shape[0]
    out = np.empty((b, s.k), np.float32)
    for j in range(s.k):
        pts = s.light_points(np.full(b, j), st.random((b, 2)))
        out[:, j] = s.visibility(pos, pts)
    return out


def train_batch(s: SceneArrays, seed: int, frame: int, step: int = 0, n_world=4096, n_screen=4096):
    key = (seed, frame, step)
    world = world_samples(s, n_world, Stream(*key, "world-samples"))
    screen = screen_samples(s, n_screen, Stream(*key, "screen-samples"))
    pos = np.concatenate([world, screen])
    return pos, targets(s, pos, Stream(*key, "targets"))


# ---------------------------------------------------------------------------
# Light selection: sampling.py:27-30, 74-85, 184-218
# ---------------------------------------------------------------------------

def wrs_select(w: np.ndarray, key: int, offset: int = 0):
    """Sequential FP64 streaming WRS; draw for (p, k) is offset + p*K + k."""
    w = np.asarray(w, np.float64)
    p, k = w.shape
    u = uniform_at(key, offset + np.arange(p * k)).reshape(p, k)
    s = np.zeros(p)
    sel = np.full(p, -1, np.int64)
    wsel = np.zeros(p)
    for j in range(k):
        s = s + w[:, j]
        take = u[:, j] * s < w[:, j]
        sel = np.where(take, j, sel)
        wsel = np.where(take, w[:, j], wsel)
    return sel, wsel, s


def nls_sample(s: SceneArrays, vis: np.ndarray, lum: np.ndarray, key: int, offset: int = 0,
               floor: float | None = 0.001, p_total: int | None = None, p_first: int = 0):
    """ids, points, W for pixels p_first.. of a P_total-pixel frame.

    Draw layout (sampling.py:194-205): WRS uses offset + p*K + k, the light
    point uses offset + P*K + 2p + {0,1} with P the frame's pixel count."""
    v = np.asarray(vis, np.float64)
    v = np.maximum(v, floor) if floor and floor > 0.0 else np.maximum(v, 0.0)
    w = v * lum
    p, k = w.shape
    ptot = p if p_total is None else p_total
    sel, wsel, wsum = wrs_select(w, key, offset + p_first * k)
    big_w = np.where(sel >= 0, wsum / np.where(wsel > 0, wsel, 1.0), 0.0)
    gp = p_first + np.arange(p)
    u = np.stack([uniform_at(key, offset + ptot * k + 2 * gp),
                  uniform_at(key, offset + ptot * k + 2 * gp + 1)], axis=1)
    return sel, s.light_points(sel, u), big_w


def neural_di(s: SceneArrays, vis: np.ndarray, factor: np.ndarray, albedo: np.ndarray):
    return ((np.asarray(vis, np.float64) * factor) @ s.lt_radiance) * albedo / np.pi


# ---------------------------------------------------------------------------
# Shading pass 5: render.py:220-246
# ---------------------------------------------------------------------------

def _dot3(a, b):
    """np.einsum("pc,pc->p") as numpy 2.3 evaluates it for c = 3: (a0 b0 + a2 b2) + a1 b1
    (pinned by tests/golden/shade.npz, which the reference's own einsum produced)."""
    return (a[:, 0] * b[:, 0] + a[:, 2] * b[:, 2]) + a[:, 1] * b[:, 1]


def shade(s: SceneArrays, pos, nrm, alb, ids, pts, big_w):              # render.py:220-246
    """One-shadow-ray estimate per row: albedo/pi * L_e * G * V * area * W."""
    pos, nrm, alb, pts = (np.asarray(a, np.float64) for a in (pos, nrm, alb, pts))
    ids, big_w = np.asarray(ids), np.asarray(big_w, np.float64)
    n = pos.shape[0]
    out = np.zeros((n, 3))
    live = (ids >= 0) & (big_w > 0)
    if not np.any(live):
        return out
    safe = np.maximum(ids, 0)
    w = pts - pos
    d2 = np.maximum(_dot3(w, w), 1e-24)
    w = w / np.sqrt(d2)[:, None]
    cos_x = np.maximum(0.0, _dot3(nrm, w))
    cos_y = np.maximum(0.0, -_dot3(w, s.lt_normal[safe]))
    geom = np.where(s.lt_kind[safe] == 0, cos_x * cos_y / d2 * s.lt_area[safe], cos_x / d2)
    live &= geom > 0
    if not np.any(live):
        return out
    vis = np.zeros(n)
    vis[live] = s.visibility(pos[live], pts[live])
    amp = geom * big_w * vis
    out[live] = (alb[live] / np.pi) * s.lt_radiance[safe[live]] * amp[live, None]
    return out


# ---------------------------------------------------------------------------
# Clustered NVC: training.py:121-128, sampling.py:302-352
# ---------------------------------------------------------------------------

def bounded_ints(key: int, start: int, count: int, n: int, pending=None):
    """numpy Generator.integers(0, n, size=count) with the stream at 64-bit output
    `start`: Lemire's bounded draw (with its rare rejection loop) on 32-bit draws.
    A 32-bit draw is the low half of a fresh output, whose high half the bit
    generator keeps for the next 32-bit draw -- also across calls (`pending`, the
    kept half or None); 64-bit draws (random()) skip it.  Returns
    (values, 64-bit outputs consumed, pending half after the call)."""
    if n == 1:
        return np.zeros(count, np.int64), 0, pending
    out = np.empty(count, np.int64)
    thresh = ((1 << 32) - n) % n
    words = raw_at(key, np.arange(start, start + (count + 1) // 2 + 8, dtype=np.uint64))
    used = 0

    def next32():
        nonlocal used, words, pending
        if pending is not None:
            v, pending = pending, None
            return v
        if used >= words.size:
            words = np.concatenate([words, raw_at(key, np.arange(start + words.size, start + words.size + 64,
                                                                 dtype=np.uint64))])
        w = int(words[used])
        used += 1
        pending = w >> 32
        return w & 0xFFFFFFFF

    for i in range(count):
        m = next32() * n
        while (m & 0xFFFFFFFF) < thresh:
            m = next32() * n
        out[i] = m >> 32
    return out, used, pending


def cluster_targets(s: SceneArrays, pos: np.ndarray, sizes, members, key: int) -> np.ndarray:
    """compute_visibility_targets(clusters=...) (training.py:121-128): per cluster a
    uniform member (integers) then its light point (random((b,2)))."""
    b = pos.shape[0]
    off = np.concatenate([[0], np.cumsum(sizes)])
    out = np.empty((b, len(sizes)), np.float32)
    st, pending = 0, None
    for j, size in enumerate(sizes):
        mem = np.asarray(members[off[j]:off[j + 1]])
        pick, used, pending = bounded_ints(key, st, b, int(size), pending)
        st += used
        u = uniform_at(key, st + np.arange(2 * b)).reshape(b, 2)
        st += 2 * b
        out[:, j] = s.visibility(pos, s.light_points(mem[pick], u))
    return out


def matmul3(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    """(r,3)@(3,c) in float64 with the reference's BLAS rounding (orc_dot3_fma)."""
    r, c = a.shape[0], b.shape[1]
    aa = np.ascontiguousarray(np.repeat(a, c, axis=0))
    bb = np.ascontiguousarray(np.tile(b.T, (r, 1)))
    out = np.empty(r * c)
    lib().orc_dot3_fma(ctypes.c_int64(r * c), _p(aa), _p(bb), ctypes.c_int32(int(r == 1 or c == 1)), _p(out))
    return out.reshape(r, c)


def clustered_sample(s: SceneArrays, vis: np.ndarray, factor: np.ndarray, albedo: np.ndarray, sizes, members,
                     key: int, offset: int = 0, floor: float | None = 0.001):
    """clustered_sample_batch (sampling.py:302-352): WRS over the clamped cluster
    visibilities, then per cluster (ascending) a WRS over its member lights with
    weights phat / p_src on the continuing stream, then the light points.
    factor: (P, K) unshadowed factors."""
    luma = np.array([0.2126, 0.7152, 0.0722])
    vis = np.asarray(vis, np.float64)
    p, m = vis.shape
    cw = np.maximum(vis, floor) if floor and floor > 0.0 else np.maximum(vis, 0.0)
    c_idx, c_w, c_sum = wrs_select(cw, key, offset)
    pos_draw = offset + p * m
    off = np.concatenate([[0], np.cumsum(sizes)])
    ids = np.full(p, -1, np.int64)
    big_w = np.zeros(p)
    for j in range(m):
        rows = np.flatnonzero(c_idx == j)
        if rows.size == 0:
            continue
        mem = np.asarray(members[off[j]:off[j + 1]])
        my = mem.size
        f = factor[np.ix_(rows, mem)]
        scale = matmul3(albedo[rows], luma[:, None] * s.lt_radiance[mem].T) / np.pi
        phat = f * scale
        p_src = m * (c_w[rows] / c_sum[rows]) / my
        w2 = phat / p_src[:, None]
        sel, _, w2_sum = wrs_select(w2, key, pos_draw)
        pos_draw += rows.size * my
        ok = sel >= 0
        rr = rows[ok]
        ids[rr] = mem[sel[ok]]
        big_w[rr] = m * w2_sum[ok] / (my * phat[ok, sel[ok]])
    u = uniform_at(key, pos_draw + np.arange(2 * p)).reshape(p, 2)
    return ids, s.light_points(ids, u), big_w
