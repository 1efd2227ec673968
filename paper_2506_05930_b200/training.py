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

import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from . import rng as rngmod
from .cache import MODE_CLUSTERS, MODE_LIGHTS, MODE_RADIANCE
from .clusters import pack_clusters
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


class BatchBuffers:
    """Device buffers for one training batch (reused across frames)."""

    def __init__(self, n_world: int, n_screen: int, k: int, device, n_shards: int = 1):
        import torch
        total = n_world + n_screen
        self.n_world, self.n_screen = n_world, n_screen
        self.pos = torch.zeros((max(total, 1), 3), dtype=torch.float64, device=device)
        self.tgt = torch.zeros((max(total // n_shards + 1, 1), k), dtype=torch.float32, device=device)
        self.n_rows = torch.zeros(1, dtype=torch.int64, device=device)
        ws = _lib.load().nvc_batch_workspace_bytes(n_world, n_screen)
        self.ws = torch.zeros(ws, dtype=torch.uint8, device=device)
        self.loss = torch.zeros(2, dtype=torch.float64, device=device)   # [sum, mean] (nvc_train_grads)


def _cluster_tables(clusters, device):
    """(c_off, c_mem) int32 device tensors of a ClusterSet, cached on it per device."""
    import torch
    cache = clusters.__dict__.setdefault("_nvc_dev", {})
    if device not in cache:
        off, flat = pack_clusters(clusters)
        cache[device] = (torch.from_numpy(off).to(device), torch.from_numpy(flat).to(device))
    return cache[device]


def _cluster_targets(ds, key, pos, n_rows, b_max, shard, n_shards, clusters, tgt, ws=None, offset=0, kept=-1):
    """nvc_cluster_targets; returns the workspace (its state block: stream position after the call)."""
    import torch
    c_off, c_mem = _cluster_tables(clusters, pos.device)
    need = _lib.load().nvc_cluster_workspace_bytes(b_max, clusters.m)
    if ws is None or ws.numel() < need:
        ws = torch.empty(need, dtype=torch.uint8, device=pos.device)
    _lib.call("nvc_cluster_targets", ds.struct, key, offset, kept, pos.data_ptr(), n_rows.data_ptr(), b_max, shard,
              n_shards, clusters.m, c_off.data_ptr(), c_mem.data_ptr(), tgt.data_ptr(), ws.data_ptr(),
              _lib.stream_ptr())
    return ws


def gen_batch_device(scene, camera, bufs: BatchBuffers, seed: int, frame: int, step: int = 0,
                     shard: int = 0, n_shards: int = 1, targets: bool = True, clusters=None) -> BatchBuffers:
    """One training batch on the device (training.py:176-195); with ``clusters`` the
    targets are cluster visibilities (training.py:121-128)."""
    ds = device_scene(scene, bufs.pos.device)
    cam = camera_struct(camera)
    key = (seed, frame, step)
    light_tgt = targets and clusters is None
    _lib.call("nvc_gen_train_batch", ds.struct, cam, rngmod.stream_key(*key, rngmod.WORLD_SAMPLES),
              rngmod.stream_key(*key, rngmod.SCREEN_SAMPLES), rngmod.stream_key(*key, rngmod.TARGETS), 0, 0,
              bufs.n_world, bufs.n_screen, shard, n_shards, bufs.pos.data_ptr(),
              bufs.tgt.data_ptr() if light_tgt else None, bufs.n_rows.data_ptr(), bufs.ws.data_ptr(),
              _lib.stream_ptr())
    if targets and clusters is not None:
        bufs.cws = _cluster_targets(ds, rngmod.stream_key(*key, rngmod.TARGETS), bufs.pos, bufs.n_rows,
                                    bufs.n_world + bufs.n_screen, shard, n_shards, clusters, bufs.tgt,
                                    getattr(bufs, "cws", None))
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
    ws = torch.zeros(_lib.load().nvc_batch_workspace_bytes(n, 0), dtype=torch.uint8, device=ds.device)
    key, off = rngmod.position(rng)            # any stream position: uniform((n,3)) draws off + 3i + c
    _lib.call("nvc_gen_train_batch", ds.struct, camera_struct(scene.camera), key, 0, 0, off, 0, n, 0, 0, 1,
              pos.data_ptr(), None, nr.data_ptr(), ws.data_ptr(), _lib.stream_ptr())
    rngmod.advance(rng, 3 * n)
    return pos.cpu().numpy()


def gen_screen_hits(scene, camera, n: int, rng):
    """training.py:67-94: primary-ray hits through uniformly random screen points,
    misses redrawn for up to SCREEN_RETRY_ROUNDS rounds (the batch may come back
    short).  Returns (positions, normals, albedos, is_light).  Each round draws sx
    then sy from ``rng`` exactly as the reference does; the rays are traced by
    nvc_primary_hits (k_gbuffer's screen-point mode)."""
    torch = _lib.require_cuda()
    ds = device_scene(scene)
    dev = ds.device
    cam = camera_struct(camera)
    parts = ([], [], [], [])
    want = int(n)
    for _ in range(SCREEN_RETRY_ROUNDS + 1):
        if want == 0:
            break
        sx = rng.random(want) * camera.width
        sy = rng.random(want) * camera.height
        sxy = torch.from_numpy(np.ascontiguousarray(np.stack([sx, sy], 1))).to(dev)
        pos, nrm, alb = (torch.empty((want, 3), dtype=torch.float64, device=dev) for _ in range(3))
        hit = torch.empty(want, dtype=torch.uint8, device=dev)
        lid = torch.empty(want, dtype=torch.int32, device=dev)
        _lib.call("nvc_primary_hits", ds.struct, cam, sxy.data_ptr(), want, pos.data_ptr(), nrm.data_ptr(),
                  alb.data_ptr(), hit.data_ptr(), lid.data_ptr(), _lib.stream_ptr())
        h = hit.bool()
        for lst, t in zip(parts, (pos[h], nrm[h], alb[h], lid[h] >= 0)):
            lst.append(t)
        want -= int(h.sum().item())
    if not parts[0]:
        return np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 3)), np.zeros(0, dtype=bool)
    return tuple(torch.cat(lst).cpu().numpy() for lst in parts)


def gen_screen_samples(scene, camera, n: int, rng) -> np.ndarray:
    """Primary-ray hit points, <= 9 rounds of redraws (training.py:67-100)."""
    import torch
    _lib.require_cuda()
    if n == 0:
        return np.zeros((0, 3))
    ds = device_scene(scene)
    bufs = BatchBuffers(0, n, ds.n_lights, ds.device)
    key, off = rngmod.position(rng)            # any stream position; rounds draw sx then sy from there
    _lib.call("nvc_gen_train_batch", ds.struct, camera_struct(camera), 0, key, 0, 0, off, 0, n, 0, 1,
              bufs.pos.data_ptr(), None, bufs.n_rows.data_ptr(), bufs.ws.data_ptr(), _lib.stream_ptr())
    b = int(bufs.n_rows.item())
    end = int(bufs.ws[16:24].view(torch.int64).item())
    rngmod.advance(rng, end - off)             # leave the stream where the reference's rounds do
    return bufs.pos[:b].cpu().numpy()


def compute_visibility_targets(positions, scene, rng, clusters=None) -> np.ndarray:
    """Binary shadow-ray targets, one column per light -- or per cluster, toward a
    uniform member (training.py:103-128)."""
    import torch
    _lib.require_cuda()
    ds = device_scene(scene)
    pos = torch.from_numpy(np.ascontiguousarray(positions, dtype=np.float64)).to(ds.device)
    b = pos.shape[0]
    key, start = rngmod.position(rng)          # any stream position, like the reference
    if clusters is not None:
        kept = -1
        if isinstance(rng, np.random.Generator) and rng.bit_generator.state.get("has_uint32"):
            kept = int(rng.bit_generator.state["uinteger"])
        tgt = torch.zeros((max(b, 1), clusters.m), dtype=torch.float32, device=ds.device)
        n_rows = torch.tensor([b], dtype=torch.int64, device=ds.device)
        ws = _cluster_targets(ds, key, pos, n_rows, max(b, 1), 0, 1, clusters, tgt, offset=start, kept=kept)
        off = _lib.load().nvc_cluster_state_offset(max(b, 1), clusters.m) // 8
        state = ws.view(torch.int64)[off + clusters.m: off + clusters.m + 2].cpu().numpy()
        rngmod.advance(rng, int(state[0]) - start)
        if isinstance(rng, np.random.Generator):
            rngmod.set_kept32(rng, None if state[1] < 0 else int(state[1]))
        return tgt[:b].cpu().numpy()
    tgt = torch.empty((b, ds.n_lights), dtype=torch.float32, device=ds.device)
    _lib.call("nvc_targets", ds.struct, key, start, pos.data_ptr(), b, tgt.data_ptr(), _lib.stream_ptr())
    rngmod.advance(rng, 2 * b * ds.n_lights)
    return tgt.cpu().numpy()


class BatchPipeline:
    """Training batches generated one frame ahead on a side stream.

    A batch depends only on (seed, frame, step) and the scene -- never on the
    model -- so batch f+1 (primary rays, FP64 shadow rays: latency- and
    FP64-bound kernels) can run while frame f trains and queries (mostly
    FP32/INT/tensor work).  Two buffers alternate; events order the side
    stream against the consumer.  One optimizer step per frame (cfg.steps == 1).
    """

    def __init__(self, scene, camera, cfg: TrainFrameConfig, k: int, device, shard: int = 0, n_shards: int = 1,
                 cache=None, clusters=None):
        import torch

        from .cache import GradExchange
        if cfg.steps != 1:
            raise ValueError("BatchPipeline prefetches one batch per frame (cfg.steps == 1)")
        self.scene, self.camera, self.cfg, self.shard, self.n_shards = scene, camera, cfg, shard, n_shards
        self.clusters = clusters
        self.bufs = [BatchBuffers(cfg.n_world, cfg.n_screen, k, device, n_shards) for _ in range(2)]
        # data parallel: the entry list of the gradient exchange depends only on the
        # batch positions, so it is built here too, off the critical path (one per buffer)
        self.ex = None
        if cache is not None and n_shards > 1 and not cache.compact:
            self.ex = [GradExchange(cache, cfg.n_world + cfg.n_screen) for _ in range(2)]
        # the batch chain (screen rays -> compaction -> shadow rays) is latency-bound:
        # give it priority so it completes within the frame it overlaps
        self.side = torch.cuda.Stream(device, priority=int(os.environ.get("NVC_BATCH_PRIORITY", "-2")))
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        cur = torch.cuda.current_stream(device)
        for e in self.free:
            e.record(cur)
        self.pending = [None, None]       # frame whose batch each buffer holds / will hold
        self.early = os.environ.get("NVC_BATCH_EARLY", "1") == "1"

    def _launch(self, frame: int) -> None:
        import torch
        b = frame % 2
        with torch.cuda.stream(self.side):
            self.side.wait_event(self.free[b])          # the previous frame on this buffer has trained
            gen_batch_device(self.scene, self.camera, self.bufs[b], self.cfg.seed, frame, 0, self.shard,
                             self.n_shards, clusters=self.clusters)
            if self.ex is not None:
                self.ex[b].index(self.bufs[b].pos, self.bufs[b].n_rows)
            self.ready[b].record(self.side)
        self.pending[b] = frame

    def take(self, frame: int) -> BatchBuffers:
        """The batch of `frame` (ready on the current stream)."""
        import torch
        b = frame % 2
        if self.pending[b] != frame:
            self._launch(frame)
        self.pending[b] = None            # consumed: the buffer is rewritten only after release()
        torch.cuda.current_stream().wait_event(self.ready[b])
        if self.early and self.pending[(frame + 1) % 2] != frame + 1:
            self._launch(frame + 1)
        return self.bufs[b]

    def exchange_for(self, bufs: BatchBuffers):
        """The GradExchange indexed for `bufs` (None if the pipeline does not build one)."""
        return None if self.ex is None else self.ex[self.bufs.index(bufs)]

    def release(self, bufs: BatchBuffers, frame: int) -> None:
        """`bufs` is consumed; start frame+1's batch (it overlaps this frame's query)."""
        import torch
        self.free[self.bufs.index(bufs)].record(torch.cuda.current_stream())
        if not self.early and self.pending[(frame + 1) % 2] != frame + 1:
            # gate the side stream on the end of this frame's training so the batch
            # chain runs under the query, not under the train step
            self.free[(frame + 1) % 2].record(torch.cuda.current_stream())
            self._launch(frame + 1)


def _check_cache(cache, cfg, clusters=None):
    if cache.mode == MODE_CLUSTERS and clusters is None:
        raise ValueError("cluster-mode cache needs a ClusterSet")
    if cache.mode == MODE_CLUSTERS and cache.output_dim != clusters.m:
        raise ValueError(f"cache has {cache.output_dim} outputs, the ClusterSet {clusters.m} clusters")
    if cache.mode == MODE_RADIANCE:
        raise NotImplementedError("the NRC radiance baseline is out of scope (SURVEY §2)")
    if cfg.surface_samples:
        raise NotImplementedError("surface_samples is off by default and not on the hot path")


def train_frame_device(scene, camera, cache, cfg: TrainFrameConfig, frame: int = 0,
                       bufs: BatchBuffers | None = None, shard: int = 0, n_shards: int = 1, comm=None,
                       pipeline: BatchPipeline | None = None, clusters=None):
    """Asynchronous frame training: returns the last step's loss as a CUDA tensor.

    With ``n_shards > 1`` every rank builds the same global batch, computes the
    targets/gradients of its row shard and ``comm(buffer, loss)`` (a sum
    allreduce of the compact GradExchange buffer and the loss) runs before the
    identical Adam update.  With ``pipeline`` the
    batch comes from (and the next one is started on) a BatchPipeline."""
    clusters = clusters if cache.mode == MODE_CLUSTERS else None
    _check_cache(cache, cfg, clusters)
    if pipeline is not None:
        if (pipeline.clusters is None) != (clusters is None):
            raise ValueError("the BatchPipeline and the cache disagree on cluster mode")
        bufs = pipeline.take(frame)
    elif bufs is None:
        bufs = BatchBuffers(cfg.n_world, cfg.n_screen, cache.output_dim, cache.device, n_shards)
    loss = None
    b_max = bufs.n_world + bufs.n_screen
    for step in range(cfg.steps):
        if pipeline is None:
            gen_batch_device(scene, camera, bufs, cfg.seed, frame, step, shard, n_shards, clusters=clusters)
        if bufs.n_world == 0 and int(bufs.n_rows.item()) == 0:
            continue    # training.py:196-197: an empty batch (all screen rays missed) skips the update
        ex = None
        if comm is not None:
            ex = pipeline.exchange_for(bufs) if pipeline is not None else None
            if ex is None:
                ex = cache.exchange(b_max)
                if not cache.compact:    # dense mode: list the global batch's entries
                    ex.index(bufs.pos, bufs.n_rows)
        cache.accumulate_grads(bufs.pos, bufs.tgt, b_max=b_max, b_dev=bufs.n_rows,
                               shard=shard, n_shards=n_shards, loss_out=bufs.loss)
        if ex is not None:
            ex.allreduce(comm, bufs.loss)
        cache.apply_adam()
        loss = bufs.loss[1]
    if pipeline is not None:
        pipeline.release(bufs, frame)
    return loss, bufs


def train_frame(scene, camera, cache, cfg: TrainFrameConfig, frame: int = 0, clusters=None) -> float:
    """Generate a fresh batch and run the configured optimizer steps; returns
    the last step's batch loss (training.py:166-199)."""
    clusters = clusters if cache.mode == MODE_CLUSTERS else None
    _check_cache(cache, cfg, clusters)
    bufs = BatchBuffers(cfg.n_world, cfg.n_screen, cache.output_dim, cache.device)
    loss = 0.0
    for step in range(cfg.steps):
        gen_batch_device(scene, camera, bufs, cfg.seed, frame, step, clusters=clusters)
        b = int(bufs.n_rows.item())
        if b == 0:            # training.py:196-197: empty batch -> no update
            continue
        cache.accumulate_grads(bufs.pos, bufs.tgt, b_max=b, shard=0, n_shards=1, loss_out=bufs.loss)
        cache.apply_adam()
        loss = float(bufs.loss[1].item())
    return loss


__all__ = ["TrainFrameConfig", "train_frame", "train_frame_device", "gen_world_samples",
           "gen_screen_samples", "compute_visibility_targets", "BatchBuffers", "gen_batch_device",
           "MODE_LIGHTS"]
