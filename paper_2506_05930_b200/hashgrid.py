"""Hash-grid configuration (host) and the device encoder entry point.

Mirrors ``viscache.hashgrid`` (hashgrid.py:22-164): same defaults, same
validation, same per-level resolution/dense rule -- the resolutions are
computed here with the reference's float expression and handed to the CUDA
kernels, so level 9 of the default growth stays 511 exactly as in the
reference.  Addressing (dense vs spatial hash with modular-add primes) and
the trilinear blend run on the GPU (csrc/common.cuh, csrc/model.cu).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib

HASH_PRIMES = (1, 2654435761, 805459861)
DEFAULT_LEVELS = 10
DEFAULT_BASE_RESOLUTION = 16
DEFAULT_FEATURES = 4
DEFAULT_TABLE_SIZE = 1 << 14
DEFAULT_SCALE = (512.0 / 16.0) ** (1.0 / 9.0)
FEATURE_INIT_SCALE = 1e-4


@dataclass
class HashGridConfig:
    levels: int = DEFAULT_LEVELS
    base_resolution: int = DEFAULT_BASE_RESOLUTION
    per_level_scale: float = DEFAULT_SCALE
    features_per_level: int = DEFAULT_FEATURES
    table_size: int = DEFAULT_TABLE_SIZE
    aabb_min: np.ndarray = field(default_factory=lambda: np.zeros(3))
    aabb_max: np.ndarray = field(default_factory=lambda: np.ones(3))

    def __post_init__(self):
        if min(self.levels, self.base_resolution, self.features_per_level) < 1:
            raise ValueError("levels, base_resolution, features_per_level must be >= 1")
        if not self.per_level_scale > 1.0:
            raise ValueError("per_level_scale must be > 1")
        t = int(self.table_size)
        if t < 1 or (t & (t - 1)) != 0:
            raise ValueError("table_size must be a power of two")
        if self.levels > _lib.MAX_LEVELS:
            raise ValueError(f"at most {_lib.MAX_LEVELS} levels are supported")
        self.aabb_min = np.asarray(self.aabb_min, dtype=np.float64)
        self.aabb_max = np.asarray(self.aabb_max, dtype=np.float64)

    @property
    def output_dim(self) -> int:
        return self.levels * self.features_per_level

    @property
    def param_count(self) -> int:
        return self.levels * self.table_size * self.features_per_level

    def resolution(self, level: int) -> int:
        return int(np.floor(self.base_resolution * self.per_level_scale ** level))

    def dense(self, level: int) -> bool:
        verts = self.resolution(level) + 1
        return verts ** 3 <= self.table_size

    def span(self) -> np.ndarray:
        return np.maximum(self.aabb_max - self.aabb_min, 1e-12)


def clustered_config(**kw) -> HashGridConfig:
    """Coarser preset for cluster outputs (hashgrid.py:68-72)."""
    kw.setdefault("levels", 8)
    kw.setdefault("base_resolution", 2)
    return HashGridConfig(**kw)


def init_table(cfg: HashGridConfig, gen: np.random.Generator, dtype=np.float32) -> np.ndarray:
    """U(-1e-4, 1e-4) feature table drawn from the init stream (hashgrid.py:75-79)."""
    shape = (cfg.levels, cfg.table_size, cfg.features_per_level)
    return gen.uniform(-FEATURE_INIT_SCALE, FEATURE_INIT_SCALE, shape).astype(dtype)


def encode_batch(positions, cache, with_ctx: bool = False):
    """Device encoder on the cache's f32 master table (exact reference rounding).

    Returns features (B, L*F) float32 numpy; with ``with_ctx`` also the
    per-level corner indices (B, L, 8) int32 and FP64 weights (B, L, 8)."""
    return cache.encode(positions, with_ctx=with_ctx)


# ---------------------------------------------------------------------------
# The reference's functional encoder API (hashgrid.py:75-164), on the device
# kernels: nvc_encode (exact FP64 index/weight math, sequential FP32 blend =
# einsum) and nvc_grid_scatter (np.add.at order).  Table and upstream must be
# float32 (the device encoder's master precision).
# ---------------------------------------------------------------------------

def init_params(cfg: HashGridConfig, rng: np.random.Generator, dtype=np.float32) -> np.ndarray:
    """hashgrid.py:75-79."""
    return init_table(cfg, rng, dtype)


def spatial_hash(coords, table_size: int):
    """hashgrid.py:82-87: (x*1 + y*2654435761 + z*805459861) & (T-1) -- modular add,
    the index arithmetic k_encode performs in uint32 (host helper for callers)."""
    c = np.asarray(coords, dtype=np.int64)
    h = c[..., 0] * HASH_PRIMES[0] + c[..., 1] * HASH_PRIMES[1] + c[..., 2] * HASH_PRIMES[2]
    return h & (table_size - 1)


_GRID_CACHES: dict = {}


def _grid_cache(cfg: HashGridConfig):
    """A device model holding cfg's table (reused per grid shape/AABB)."""
    import torch
    from .cache import MODE_LIGHTS, VisibilityCache
    key = (cfg.levels, cfg.table_size, cfg.features_per_level, cfg.base_resolution, cfg.per_level_scale,
           tuple(np.asarray(cfg.aabb_min, np.float64)), tuple(np.asarray(cfg.aabb_max, np.float64)),
           torch.cuda.current_device())
    c = _GRID_CACHES.get(key)
    if c is None:
        c = _GRID_CACHES[key] = VisibilityCache(MODE_LIGHTS, 8, cfg)
    return c


def _encode_functional(pos, cfg: HashGridConfig, params):
    import torch
    _lib.require_cuda()
    params = np.asarray(params)
    shape = (cfg.levels, cfg.table_size, cfg.features_per_level)
    if params.shape != shape:
        raise ValueError(f"params must be {shape}, got {params.shape}")
    if params.dtype != np.float32:
        raise ValueError("the CUDA encoder reads a float32 feature table")
    c = _grid_cache(cfg)
    c.params[:cfg.param_count].copy_(torch.from_numpy(np.ascontiguousarray(params).reshape(-1)))
    feats, idx, w = c.encode(np.atleast_2d(np.asarray(pos, dtype=np.float64)), with_ctx=True)
    ctx = [(idx[:, lvl, :].astype(np.int64), w[:, lvl, :]) for lvl in range(cfg.levels)]
    return feats, ctx


def encode_batch(pos, cfg, params=None, with_ctx: bool = False):
    """``encode_batch(pos, cfg, params)`` (hashgrid.py:117-131): features (B, L*F)
    float32 and ctx = [(idx (B,8) int64, w (B,8) float64)] per level.

    ``encode_batch(positions, cache, with_ctx=False)``: the same encoder on a
    VisibilityCache's own table (features, or features + (B,L,8) idx / w)."""
    if isinstance(cfg, HashGridConfig):
        return _encode_functional(pos, cfg, params)
    return cfg.encode(pos, with_ctx=with_ctx)


def encode(pos, cfg: HashGridConfig, params) -> np.ndarray:
    """hashgrid.py:134-137: the feature vector of one position."""
    out, _ = _encode_functional(np.asarray(pos, dtype=np.float64)[None, :], cfg, params)
    return out[0]


def grad_from_ctx(cfg: HashGridConfig, ctx, upstream, dtype=None) -> np.ndarray:
    """hashgrid.py:140-151: dense (L, T, F) table gradient, every entry the
    sequential float32 sum of float32(w * g) in (row, corner) order (np.add.at);
    bit-identical, on nvc_grid_scatter."""
    import torch
    _lib.require_cuda()
    up = np.atleast_2d(np.asarray(upstream))
    dtype = np.dtype(dtype or up.dtype)
    if dtype != np.float32 or up.dtype != np.float32:
        raise ValueError("the CUDA scatter accumulates float32 upstream gradients into a float32 table")
    b, lv = up.shape[0], len(ctx)
    if lv != cfg.levels or up.shape[1] != cfg.output_dim:
        raise ValueError("ctx / upstream do not match the grid config")
    dev = torch.device("cuda", torch.cuda.current_device())
    idx = np.stack([np.asarray(i).reshape(b, 8) for i, _ in ctx], 1).astype(np.int32)
    w = np.stack([np.asarray(x, np.float64).reshape(b, 8) for _, x in ctx], 1)
    idx_d = torch.from_numpy(np.ascontiguousarray(idx)).to(dev)
    w_d = torch.from_numpy(np.ascontiguousarray(w)).to(dev)
    up_d = torch.from_numpy(np.ascontiguousarray(up)).to(dev)
    grad = torch.zeros((cfg.levels, cfg.table_size, cfg.features_per_level), dtype=torch.float32, device=dev)
    _lib.call("nvc_grid_scatter", cfg.levels, cfg.features_per_level, cfg.table_size, idx_d.data_ptr(),
              w_d.data_ptr(), up_d.data_ptr(), b, grad.data_ptr(), _lib.stream_ptr())
    return grad.cpu().numpy()


def encode_backward(pos, cfg: HashGridConfig, params, upstream) -> np.ndarray:
    """hashgrid.py:154-164: gradient of upstream . encode(pos) w.r.t. the table."""
    _, ctx = _encode_functional(np.atleast_2d(np.asarray(pos, dtype=np.float64)), cfg, params)
    return grad_from_ctx(cfg, ctx, np.atleast_2d(upstream), dtype=np.asarray(params).dtype)
