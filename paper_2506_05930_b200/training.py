"""Per-frame training batches and the online train step: drop-in for
``viscache.training`` (training.py:21-199), light mode.

A batch is generated entirely on the GPU (``nvc_gen_train_batch``): world
samples from the (seed, frame, step, "world-samples") stream, screen samples
from primary rays with up to 9 order-preserving retry rounds, and one FP64
shadow ray per (position, light) -- bit-identical to the reference.  The
train step then runs ``nvc_train_grads`` (fixed-point deterministic scatter)
and the fused dense Adam without a host round trip; only the returned loss
(a Python float, as in the reference) synchronises.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from . import rng as rngmod
from .cache import MODE_CLUSTERS, MODE_LIGHTS, MODE_RADIANCE
from .scene import camera_struct, device_scene

SCREEN_RETRY_ROUNDS = 8


@dataclass
class TrainFrameConfig:
    n_world: int = 4096
    n_screen: int = 4096
    steps: int = 1
    surface_samples: bool = False
    seed: int = 0

    @property
    def batch_size(self) -> int:
        return self.n_world + self.n_screen

    @classmethod
    def clustered(cls, **kw) -> "TrainFrameConfig":
        kw.setdefault("n_world", 24576)
        kw.setdefault("n_screen", 24576)
        return cls(**kw)


def _fresh_key(g) -> int:
    key, off = rngmod.position(g)
    if off != 0:
        raise ValueError("training-batch streams must be fresh (as train_frame creates them)")
    return key


class BatchBuffers:
    """Device buffers for one training batch (reused across frames)."""

    def __init__(self, n_world: int, n_screen: int, k: int, device, n_shards: int = 1):
        import torch
        total = n_world + n_screen
        self.n_world, self.n_screen = n_world, n_screen
        self.pos = torch.zeros((max(total, 1), 3), dtype=torch.float64, device=device)
        self.tgt = torch.zeros((max(total // n_shards + 1, 1), k), dtype=torch.float32, device=device)
        self.n_rows = torch.zeros(1, dtype=torch.int64, device=device)
        ws = _lib.load().nvc_batch_workspace_bytes(n_screen)
        self.ws = torch.zeros(ws, dtype=torch.uint8, device=device)
        self.loss = torch.zeros(1, dtype=torch.float64, device=device)


def gen_batch_device(scene, camera, bufs: BatchBuffers, seed: int, frame: int, step: int = 0,
                     shard: int = 0, n_shards: int = 1, targets: bool = True) -> BatchBuffers:
    ds = device_scene(scene, bufs.pos.device)
    cam = camera_struct(camera)
    key = (seed, frame, step)
    _lib.call("nvc_gen_train_batch", ds.struct, cam, rngmod.stream_key(*key, rngmod.WORLD_SAMPLES),
              rngmod.stream_key(*key, rngmod.SCREEN_SAMPLES), rngmod.stream_key(*key, rngmod.TARGETS),
              bufs.n_world, bufs.n_screen, shard, n_shards, bufs.pos.data_ptr(),
              bufs.tgt.data_ptr() if targets else None, bufs.n_rows.data_ptr(), bufs.ws.data_ptr(),
              _lib.stream_ptr())
    return bufs


def gen_world_samples(scene, n: int, rng) -> np.ndarray:
    """n points uniform in the scene AABB (training.py:44-48)."""
    import torch
    _lib.require_cuda()
    if n == 0:
        return np.zeros((0, 3))
    ds = device_scene(scene)
    pos = torch.zeros((n, 3), dtype=torch.float64, device=ds.device)
    nr = torch.zeros(1, dtype=torch.int64, device=ds.device)
    ws = torch.zeros(_lib.load().nvc_batch_workspace_bytes(0), dtype=torch.uint8, device=ds.device)
    _lib.call("nvc_gen_train_batch", ds.struct, camera_struct(scene.camera), _fresh_key(rng), 0, 0, n, 0, 0, 1,
              pos.data_ptr(), None, nr.data_ptr(), ws.data_ptr(), _lib.stream_ptr())
    rngmod.advance(rng, 3 * n)
    return pos.cpu().numpy()


def gen_screen_samples(scene, camera, n: int, rng) -> np.ndarray:
    """Primary-ray hit points, <= 9 rounds of redraws (training.py:67-100)."""
    import torch
    _lib.require_cuda()
    if n == 0:
        return np.zeros((0, 3))
    ds = device_scene(scene)
    bufs = BatchBuffers(0, n, ds.n_lights, ds.device)
    _lib.call("nvc_gen_train_batch", ds.struct, camera_struct(camera), 0, _fresh_key(rng), 0, 0, n, 0, 1,
              bufs.pos.data_ptr(), None, bufs.n_rows.data_ptr(), bufs.ws.data_ptr(), _lib.stream_ptr())
    b = int(bufs.n_rows.item())
    return bufs.pos[:b].cpu().numpy()


def compute_visibility_targets(positions, scene, rng, clusters=None) -> np.ndarray:
    """Binary shadow-ray targets, one column per light (training.py:103-120)."""
    import torch
    if clusters is not None:
        raise NotImplementedError("cluster targets are outside this build's hot path (SURVEY §8(f))")
    _lib.require_cuda()
    ds = device_scene(scene)
    pos = torch.from_numpy(np.ascontiguousarray(positions, dtype=np.float64)).to(ds.device)
    b = pos.shape[0]
    tgt = torch.empty((b, ds.n_lights), dtype=torch.float32, device=ds.device)
    _lib.call("nvc_targets", ds.struct, _fresh_key(rng), pos.data_ptr(), b, tgt.data_ptr(), _lib.stream_ptr())
    rngmod.advance(rng, 2 * b * ds.n_lights)
    return tgt.cpu().numpy()


def _check_cache(cache, cfg):
    if cache.mode == MODE_CLUSTERS:
        raise NotImplementedError("clustered NVC is outside this build's hot path (SURVEY §8(f))")
    if cache.mode == MODE_RADIANCE:
        raise NotImplementedError("the NRC radiance baseline is out of scope (SURVEY §2)")
    if cfg.surface_samples:
        raise NotImplementedError("surface_samples is off by default and not on the hot path")


def train_frame_device(scene, camera, cache, cfg: TrainFrameConfig, frame: int = 0,
                       bufs: BatchBuffers | None = None, shard: int = 0, n_shards: int = 1, comm=None):
    """Asynchronous frame training: returns the last step's loss as a CUDA tensor.

    With ``n_shards > 1`` every rank builds the same global batch, computes the
    targets/gradients of its row shard and ``comm(grad_fx, loss)`` (an
    allreduce) runs before the identical Adam update."""
    _check_cache(cache, cfg)
    if bufs is None:
        bufs = BatchBuffers(cfg.n_world, cfg.n_screen, cache.output_dim, cache.device, n_shards)
    loss = None
    for step in range(cfg.steps):
        gen_batch_device(scene, camera, bufs, cfg.seed, frame, step, shard, n_shards)
        bufs.loss.zero_()
        cache.accumulate_grads(bufs.pos, bufs.tgt, b_max=bufs.n_world + bufs.n_screen, b_dev=bufs.n_rows,
                               shard=shard, n_shards=n_shards, loss_out=bufs.loss)
        if comm is not None:
            comm(cache.grad_fx, bufs.loss)
        cache.apply_adam()
        loss = bufs.loss[0] / bufs.n_rows[0].to(bufs.loss.dtype)
    return loss, bufs


def train_frame(scene, camera, cache, cfg: TrainFrameConfig, frame: int = 0, clusters=None) -> float:
    """Generate a fresh batch and run the configured optimizer steps; returns
    the last step's batch loss (training.py:166-199)."""
    if cache.mode == MODE_CLUSTERS and clusters is None:
        raise ValueError("cluster-mode cache needs a ClusterSet")
    _check_cache(cache, cfg)
    bufs = BatchBuffers(cfg.n_world, cfg.n_screen, cache.output_dim, cache.device)
    loss = 0.0
    for step in range(cfg.steps):
        gen_batch_device(scene, camera, bufs, cfg.seed, frame, step)
        b = int(bufs.n_rows.item())
        if b == 0:            # training.py:196-197: empty batch -> no update
            continue
        bufs.loss.zero_()
        cache.accumulate_grads(bufs.pos, bufs.tgt, b_max=b, shard=0, n_shards=1, loss_out=bufs.loss)
        cache.apply_adam()
        loss = float(bufs.loss.item()) / b
    return loss


__all__ = ["TrainFrameConfig", "train_frame", "train_frame_device", "gen_world_samples",
           "gen_screen_samples", "compute_visibility_targets", "BatchBuffers", "gen_batch_device",
           "MODE_LIGHTS"]
