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
