"""The neural visibility cache: drop-in for ``viscache.cache`` (cache.py:25-139).

State lives in HBM as one flat f32 parameter vector in the reference's
``_param_dict`` order (grid, w0, b0, w1, b1, ...) plus Adam moments, an int64
fixed-point gradient accumulator (zero except where this step's samples
touched the table; consumed and cleared by Adam), the fp16 shadow table the query kernel gathers from, and the fp16 weights packed in
the tcgen05 core-matrix layout.  ``infer`` and ``train_step`` keep the
reference's numpy-in / numpy-out signatures; ``*_device`` variants take and
return CUDA tensors without host round trips.

Extension over the reference: ``hidden_dims`` (the reference hardcodes
(32, 32), cache.py:37-38).  Initialisation follows cache.py:41-43 for any
width: one (seed, "init-params") stream, table first, then He weights.
"""

from __future__ import annotations

import json
import struct
import weakref
from dataclasses import asdict

import numpy as np

from . import _lib
from . import rng as rngmod
from .hashgrid import HashGridConfig, clustered_config, init_table
from .mlp import LEAKY, SIGMOID, AdamState, MLPConfig, MLPParams, TrainStepConfig, he_init, lr_at

MODE_LIGHTS = "lights"
MODE_CLUSTERS = "clusters"
MODE_RADIANCE = "radiance"
SNAP_MAGIC = b"VCSNAP1\n"

PRECISION_FP32 = 0     # f32 table + f32 SIMT MLP (parity path)
PRECISION_FP16 = 1     # fp16 shadow table + tcgen05/TMEM MLP (perf path)


class GradExchange:
    """Compact data-parallel gradient exchange (nvc.h, nvc_exchange_*).

    All ranks hold the same global batch, so the hash-table entries it touches
    are the same everywhere: ``index`` lists them, ``pack`` gathers their
    fixed-point gradients (+ the MLP gradients) into ``buf``, the caller
    allreduces ``buf`` (about 1/8 of the dense accumulator at C2), ``unpack``
    writes the sums back.  Equal to the dense allreduce bit for bit."""

    def __init__(self, cache, b_max: int):
        import torch
        lib = _lib.load()
        self.cache = cache
        self.b_max = int(b_max)
        self.max_entries = int(lib.nvc_exchange_max_entries(cache.model, self.b_max))
        dev = cache.device
        if cache.compact:   # the compact gradient slots are exchanged in place
            self.ws = self.idx = self.count = self.buf = None
            return
        self.ws = torch.empty(int(lib.nvc_exchange_workspace_bytes(cache.model)), dtype=torch.uint8, device=dev)
        self.idx = torch.empty(max(self.max_entries, 1), dtype=torch.int32, device=dev)
        self.count = torch.zeros(1, dtype=torch.int64, device=dev)
        self.buf = torch.zeros(int(lib.nvc_exchange_buffer_len(cache.model, self.max_entries)), dtype=torch.int64,
                               device=dev)

    def index(self, pos, b_dev=None) -> None:
        _lib.call("nvc_exchange_index", self.cache.model, pos.data_ptr(), self.b_max, _lib.ptr(b_dev),
                  self.ws.data_ptr(), self.idx.data_ptr(), self.count.data_ptr(), _lib.stream_ptr())

    def pack(self) -> None:
        _lib.call("nvc_exchange_pack", self.cache.model, self.idx.data_ptr(), self.count.data_ptr(),
                  self.max_entries, self.buf.data_ptr(), _lib.stream_ptr())

    def unpack(self) -> None:
        _lib.call("nvc_exchange_unpack", self.cache.model, self.idx.data_ptr(), self.count.data_ptr(),
                  self.max_entries, self.buf.data_ptr(), _lib.stream_ptr())

    def allreduce(self, comm, loss) -> None:
        """Compact mode: comm(grad_c, loss) -- the compact slots ARE the exchange
        buffer.  Dense mode: pack -> comm(buf, loss) -> unpack."""
        if self.cache.grad_c is not None:
            comm(self.cache.grad_c, loss)
            return
        self.pack()
        comm(self.buf, loss)
        self.unpack()


class VisibilityCache:
    """Online-trained cache: position -> one sigmoid output per light/cluster."""

    def __init__(self, mode: str, output_dim: int, grid: HashGridConfig,
                 train: TrainStepConfig | None = None, seed: int = 0, dtype=np.float32,
                 hidden_dims=(32, 32), device=None, precision: int = PRECISION_FP16):
        if mode not in (MODE_LIGHTS, MODE_CLUSTERS, MODE_RADIANCE):
            raise ValueError(f"unknown cache mode {mode!r}")
        if np.dtype(dtype) != np.float32:
            # documented refusal (DESIGN 1): the reference's float64 mode exists to
            # calibrate tolerances on the CPU; the device path keeps f32 masters
            raise ValueError(f"dtype={np.dtype(dtype).name}: the CUDA cache keeps float32 master parameters "
                             "(the reference's float64 mode is a CPU-only calibration path)")
        torch = _lib.require_cuda()
        self.mode = mode
        self.output_dim = int(output_dim)
        self.grid_cfg = grid
        self.net_cfg = MLPConfig(input_dim=grid.output_dim, output_dim=self.output_dim,
                                 hidden_dims=tuple(hidden_dims),
                                 output_activation=LEAKY if mode == MODE_RADIANCE else SIGMOID)
        self.train_cfg = train or TrainStepConfig()
        self.dtype = np.dtype(np.float32)
        self.precision = precision
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.step = 0          # train_step count (drives lr_at)
        self.adam_t = 0        # Adam bias-correction step
        gen = rngmod.stream(seed, rngmod.INIT_PARAMS)
        table = init_table(grid, gen)
        net = he_init(self.net_cfg, gen)
        self._alloc()
        self._upload(table, net)

    # ---- state ----------------------------------------------------------
    def _offsets(self):
        offs, o = [], self.grid_cfg.param_count
        for fo, fi in self.net_cfg.layer_dims:
            offs.append((o, o + fo * fi))
            o += fo * fi + fo
        return offs, o

    def _alloc(self) -> None:
        import torch
        offs, total = self._offsets()
        self._layer_offs = offs
        self.param_count_ = total
        dev = self.device
        g = self.grid_cfg
        self.params = torch.zeros(total, dtype=torch.float32, device=dev)
        self.adam_m = torch.zeros_like(self.params)
        self.adam_v = torch.zeros_like(self.params)
        # dense int64 gradient accumulator: used only when compact gradients are off
        self.grad_fx = torch.zeros(total, dtype=torch.int64, device=dev)
        self.grad_c = None          # compact mode buffers (allocated on the first train step)
        # compact gradients (nvc.h): ~17 MB of slots instead of the 134 MB dense
        # accumulator at C2 and an in-place data-parallel exchange buffer; measured
        # slower per step on one B200 (the entry bitmap costs more than the dense
        # stream saves), so off by default
        self.compact = False
        # fp16 query table in x-pair layout (common.cuh): 2 x the grid parameters
        self.table_h = torch.zeros(2 * g.param_count, dtype=torch.float16, device=dev)
        m = _lib.NvcModel()
        m.levels, m.features, m.table_size = g.levels, g.features_per_level, g.table_size
        for level in range(g.levels):
            m.resolution[level] = g.resolution(level)
            m.dense[level] = int(g.dense(level))
        span = np.maximum(np.asarray(g.aabb_max, np.float64) - np.asarray(g.aabb_min, np.float64), 1e-12)
        for a in range(3):
            m.aabb_min[a] = float(g.aabb_min[a])
            m.span[a] = float(span[a])
        dims = self.net_cfg.dims
        if len(dims) - 1 > _lib.MAX_LAYERS:
            raise ValueError(f"at most {_lib.MAX_LAYERS} layers are supported")
        m.n_layers = len(dims) - 1
        for i, d in enumerate(dims):
            m.dims[i] = d
        m.alpha = self.net_cfg.alpha
        m.out_sigmoid = int(self.net_cfg.output_activation == SIGMOID)
        m.param_count = total
        wc = _lib.load().nvc_wpack_count(m)
        self.wpack = torch.zeros(wc, dtype=torch.int16, device=dev)
        m.wpack_count = wc
        m.params, m.adam_m, m.adam_v = (t.data_ptr() for t in (self.params, self.adam_m, self.adam_v))
        m.grad_fx = self.grad_fx.data_ptr()
        m.table_h, m.wpack = self.table_h.data_ptr(), self.wpack.data_ptr()
        self.model = m
        self._mirror = None       # host copy of `params` behind grid_params / net_params views
        self._handouts = []       # weakrefs to views a caller may still write into
        self._dirty = False       # views handed out since the last upload
        self._opt_shard = None    # sharded optimizer (set_optimizer_shard)
        self._ws = None
        self._qws = None
        self.select_done = None   # CUDA event: last off-stream NLS selection finished
        self._exchange = None
        # "pipeline": decoupled encode -> tcgen05 MLP -> selection (default);
        # "fused": the single fused kernel

    def _upload(self, table: np.ndarray, net: MLPParams) -> None:
        import torch
        flat = np.concatenate([np.asarray(table, np.float32).reshape(-1)]
                              + [x for w, b in zip(net.weights, net.biases)
                                 for x in (np.asarray(w, np.float32).reshape(-1), np.asarray(b, np.float32))])
        self.params.copy_(torch.from_numpy(flat))
        self.refresh_shadow()
        if self._mirror is not None:
            self._mirror[...] = flat

    def refresh_shadow(self, stream=None) -> None:
        _lib.call("nvc_refresh_shadow", self.model, _lib.stream_ptr(stream))

    def pin_table_in_l2(self, stream=None) -> None:
        """Keep the fp16 query table in the persisting L2 carve-out (best effort)."""
        _lib.call("nvc_l2_persist", self.table_h.data_ptr(), self.table_h.numel() * 2, _lib.stream_ptr(stream))

    @property
    def param_count(self) -> int:
        return self.param_count_

    # ---- host views of the parameters (write-through) ---------------------
    # The reference's grid_params / net_params are the live arrays Adam updates
    # in place, and callers may write into them (test_render.py:176-179).  Here
    # they are views into one host mirror of the device vector.  Once a view
    # has been handed out the mirror is "dirty": the next device op uploads it
    # (applying any caller writes), and while a view is still alive every
    # parameter update is downloaded into it.  With no view handed out (the
    # hot path) nothing is copied.
    def _views_alive(self) -> bool:
        self._handouts = [r for r in self._handouts if r() is not None]
        return bool(self._handouts)

    def _handout(self, view: np.ndarray) -> np.ndarray:
        self._handouts.append(weakref.ref(view))
        self._dirty = True
        return view

    def _host_params(self) -> np.ndarray:
        """The flat host mirror, current with the device (plus pending caller writes)."""
        if self._mirror is None:
            self._mirror = np.empty(self.param_count_, dtype=np.float32)
        elif getattr(self, "_dirty", False):
            return self._mirror
        self._mirror[...] = self.params.detach().cpu().numpy()
        return self._mirror

    def _push_views(self) -> None:
        """Before a device op reads parameters: apply caller writes to handed-out views."""
        if getattr(self, "_dirty", False):
            import torch
            self.params.copy_(torch.from_numpy(self._mirror))
            self.refresh_shadow()
            self._dirty = self._views_alive()

    def _pull_views(self) -> None:
        """After a device op changed parameters: refresh live views in place."""
        if getattr(self, "_dirty", False) and self._views_alive():
            self._mirror[...] = self.params.detach().cpu().numpy()
        elif self._mirror is not None:
            self._dirty = False

    @property
    def grid_params(self) -> np.ndarray:
        g = self.grid_cfg
        flat = self._host_params()
        return self._handout(flat[:g.param_count].reshape(g.levels, g.table_size, g.features_per_level))

    @grid_params.setter
    def grid_params(self, value) -> None:
        self._upload(value, self.net_params)

    @property
    def net_params(self) -> MLPParams:
        flat = self._host_params()
        ws, bs = [], []
        for (wo, bo), (fo, fi) in zip(self._layer_offs, self.net_cfg.layer_dims):
            ws.append(self._handout(flat[wo:wo + fo * fi].reshape(fo, fi)))
            bs.append(self._handout(flat[bo:bo + fo]))
        return MLPParams(ws, bs)

    @net_params.setter
    def net_params(self, value: MLPParams) -> None:
        self._upload(self.grid_params, value)

    def _param_dict(self) -> dict:
        return {"grid": self.grid_params, **self.net_params.as_dict()}

    def _split(self, flat: np.ndarray) -> dict:
        g = self.grid_cfg
        out = {"grid": flat[:g.param_count].reshape(g.levels, g.table_size, g.features_per_level)}
        for i, ((wo, bo), (fo, fi)) in enumerate(zip(self._layer_offs, self.net_cfg.layer_dims)):
            out[f"w{i}"] = flat[wo:wo + fo * fi].reshape(fo, fi)
            out[f"b{i}"] = flat[bo:bo + fo]
        return out

    @property
    def adam(self) -> AdamState:
        """Adam moments per parameter array and the step (reference ``cache.adam``,
        cache.py:44): a host snapshot; assign an AdamState to restore one."""
        return AdamState(m=self._split(self.adam_m.cpu().numpy()), v=self._split(self.adam_v.cpu().numpy()),
                         t=self.adam_t)

    @adam.setter
    def adam(self, state) -> None:
        import torch
        names = list(self._split(np.zeros(self.param_count_, np.float32)))
        for dst, src in ((self.adam_m, state.m), (self.adam_v, state.v)):
            flat = np.concatenate([np.asarray(src[k], np.float32).reshape(-1) for k in names])
            dst.copy_(torch.from_numpy(flat))
        self.adam_t = int(state.t)

    def adam_state(self) -> dict:
        """Adam moments and step (the reference snapshot omits these)."""
        return {"m": self.adam_m.cpu().numpy(), "v": self.adam_v.cpu().numpy(), "t": self.adam_t}

    # ---- encoder / inference --------------------------------------------
    def _pos_device(self, positions):
        import torch
        if isinstance(positions, torch.Tensor):
            if positions.device != self.device or positions.dtype != torch.float64:
                positions = positions.to(self.device, torch.float64)
            return positions.contiguous(), True
        pos = np.atleast_2d(np.asarray(positions, dtype=np.float64))
        if pos.shape[1] != 3:
            raise ValueError(f"positions must be (B, 3), got {pos.shape}")
        if not np.all(np.isfinite(pos)):
            raise ValueError("non-finite input features")
        return torch.from_numpy(np.ascontiguousarray(pos)).to(self.device), False

    def encode(self, positions, with_ctx: bool = False):
        import torch
        self._push_views()
        pos, is_dev = self._pos_device(positions)
        n = pos.shape[0]
        g = self.grid_cfg
        feats = torch.empty((n, g.output_dim), dtype=torch.float32, device=self.device)
        idx = torch.empty((n, g.levels, 8), dtype=torch.int32, device=self.device) if with_ctx else None
        w = torch.empty((n, g.levels, 8), dtype=torch.float64, device=self.device) if with_ctx else None
        _lib.call("nvc_encode", self.model, pos.data_ptr(), n, feats.data_ptr(), _lib.ptr(idx), _lib.ptr(w),
                  _lib.stream_ptr())
        if is_dev:
            return (feats, idx, w) if with_ctx else feats
        out = feats.cpu().numpy()
        return (out, idx.cpu().numpy(), w.cpu().numpy()) if with_ctx else out

    def query_workspace(self, p: int):
        """Scratch of the fp16 query pipeline for p pixels (grown on demand).

        If a selection is still running on another stream (``select_done``),
        the current stream first waits for it: it reads this workspace."""
        import torch
        self._push_views()
        if p <= 0:
            return None
        if self.select_done is not None:
            torch.cuda.current_stream().wait_event(self.select_done)
            self.select_done = None
        need = _lib.load().nvc_query_workspace_bytes(self.model, p)
        if self._qws is None or self._qws.numel() < need:
            self._qws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._qws

    def infer_device(self, pos, precision: int | None = None, out=None):
        import torch
        self._push_views()
        n = pos.shape[0]
        if out is None:
            out = torch.empty((n, self.output_dim), dtype=torch.float32, device=self.device)
        prec = self.precision if precision is None else precision
        ws = self.query_workspace(n) if prec == PRECISION_FP16 else None
        try:
            _lib.call("nvc_infer", self.model, pos.data_ptr(), n, prec, out.data_ptr(), _lib.ptr(ws),
                      _lib.stream_ptr())
        except _lib.NvcUnsupported:
            if prec != PRECISION_FP16:
                raise
            # topology the tcgen05 kernels do not cover (smem/width limits): fp32 CUDA path
            _lib.call("nvc_infer", self.model, pos.data_ptr(), n, PRECISION_FP32, out.data_ptr(), None,
                      _lib.stream_ptr())
        return out

    def infer(self, positions, precision: int | None = None):
        """Predictions for (B,3) positions, shape (B, output_dim) float32."""
        pos, is_dev = self._pos_device(positions)
        out = self.infer_device(pos, precision)
        return out if is_dev else out.cpu().numpy()

    # ---- training -------------------------------------------------------
    def _workspace(self, b: int):
        import torch
        need = _lib.load().nvc_train_workspace_bytes(self.model, b)
        if self._ws is None or self._ws.numel() < need:
            self._ws = torch.empty(need, dtype=torch.uint8, device=self.device)
        return self._ws

    def accumulate_grads(self, pos, targets, mask=None, b_max=None, b_dev=None, shard=0, n_shards=1,
                         loss_out=None):
        """Device gradient accumulation (the allreduce point for data parallelism)."""
        import torch
        self._push_views()
        b_max = int(pos.shape[0] if b_max is None else b_max)
        if loss_out is None:
            loss_out = torch.zeros(2, dtype=torch.float64, device=self.device)   # [sum, mean]
        ws = self._workspace(b_max)
        if self.compact:
            self._bind_compact(b_max)
            _lib.call("nvc_train_index", self.model, pos.data_ptr(), b_max, _lib.ptr(b_dev), _lib.stream_ptr())
        _lib.call("nvc_train_grads", self.model, pos.data_ptr(), targets.data_ptr(), _lib.ptr(mask), b_max,
                  _lib.ptr(b_dev), shard, n_shards, ws.data_ptr(), loss_out.data_ptr(), _lib.stream_ptr())
        return loss_out

    def apply_adam(self) -> None:
        lr = lr_at(self.step, self.train_cfg)
        self.adam_t += 1
        sh = self._opt_shard
        if sh is None:
            _lib.call("nvc_adam_step", self.model, self.adam_t, lr, _lib.stream_ptr())
        else:
            # sharded optimizer: this rank updates its slice of the table (+ the MLP),
            # then the slices are all-gathered and the fp16 query table rebuilt
            shard, n, gather, lo, hi, buf = sh
            _lib.call("nvc_adam_step_shard", self.model, self.adam_t, lr, shard, n, _lib.stream_ptr())
            buf[:hi - lo].copy_(self.params[lo:hi])
            gathered = gather(buf)                     # (n, span) in rank order
            for r in range(n):
                rlo, rhi = self._opt_ranges[r]
                self.params[rlo:rhi].copy_(gathered[r, :rhi - rlo])
            self.refresh_shadow()
        self.step += 1
        self._pull_views()

    def _adam_range(self, shard: int, n_shards: int):
        """[lo, hi) of the table parameters shard `shard` of n_shards updates."""
        lo, hi = _lib.ctypes.c_int64(), _lib.ctypes.c_int64()
        _lib.call("nvc_adam_shard_range", self.model, shard, n_shards, _lib.ctypes.byref(lo), _lib.ctypes.byref(hi))
        return lo.value, hi.value

    def set_optimizer_shard(self, shard: int, n_shards: int, all_gather=None) -> None:
        """Shard the optimizer over data-parallel ranks: each rank runs
        Adam on 1/n_shards of the hash-table parameters (its m/v slices are the only
        ones it keeps current) and ``all_gather(buf) -> (n_shards, len(buf))``
        collects the updated slices (e.g. torch.distributed.all_gather_into_tensor).
        The gradients must be the allreduced sum (GradExchange, dense mode).  The
        result is bit-identical to the replicated update; n_shards == 1 turns it off."""
        import torch
        if n_shards <= 1:
            self._opt_shard = None
            return
        if self.compact:
            raise ValueError("the sharded optimizer needs dense gradients (set_compact(False))")
        ranges = [self._adam_range(r, n_shards) for r in range(n_shards)]
        self._opt_ranges = ranges
        self._opt_span = max(h - l for l, h in ranges)
        lo, hi = ranges[shard]
        buf = torch.zeros(self._opt_span, dtype=torch.float32, device=self.device)
        self._opt_shard = (shard, n_shards, all_gather, lo, hi, buf)

    def _bind_compact(self, b_max: int) -> None:
        """(Re)allocate the compact-gradient buffers for batches of up to b_max rows."""
        import torch
        lib = _lib.load()
        need = int(lib.nvc_exchange_max_entries(self.model, b_max))
        if self.grad_c is not None and self.model.grad_c_entries >= need:
            return
        dev = self.device
        self.touch_bits = torch.zeros(int(lib.nvc_touch_words(self.model)), dtype=torch.int32, device=dev)
        self.touch_off = torch.zeros(int(lib.nvc_touch_off_len(self.model)), dtype=torch.int32, device=dev)
        self.grad_c = torch.zeros(int(lib.nvc_exchange_buffer_len(self.model, need)), dtype=torch.int64, device=dev)
        self.model.touch_bits = self.touch_bits.data_ptr()
        self.model.touch_off = self.touch_off.data_ptr()
        self.model.grad_c = self.grad_c.data_ptr()
        self.model.grad_c_entries = need

    def set_compact(self, on: bool) -> None:
        """Compact gradient slots (on) or the dense fixed-point accumulator (off, the
        default: measured faster on one GPU); switch only between steps."""
        self.compact = bool(on)
        if not on:
            self.model.grad_c = None
            self.grad_c = None

    def exchange(self, b_max: int) -> GradExchange:
        """The (cached) compact gradient exchange for batches of up to b_max rows."""
        if self._exchange is None or self._exchange.b_max < b_max:
            self._exchange = GradExchange(self, b_max)
        return self._exchange

    def train_step_device(self, pos, targets, mask=None, b_dev=None, b_max=None, comm=None):
        """One fused step on device tensors; returns the loss as a 0-d CUDA tensor
        (sum of per-row losses / b) without synchronising.  ``comm`` is an
        optional callable(buffer, loss) that sum-allreduces both in place; it
        receives the compact gradient exchange buffer (GradExchange)."""
        b = int(pos.shape[0] if b_max is None else b_max)
        if comm is not None and not self.compact:
            ex = self.exchange(b)
            ex.index(pos, b_dev)
        loss = self.accumulate_grads(pos, targets, mask, b_max=b_max, b_dev=b_dev)
        if comm is not None and self.compact:
            ex = self.exchange(b)
        if comm is not None:
            ex.allreduce(comm, loss)
        self.apply_adam()
        return loss[1]

    def train_step(self, positions, targets, mask=None) -> float:
        """One fused encode/forward/backward/Adam update. Returns batch loss."""
        import torch
        pos, _ = self._pos_device(positions)
        tg = torch.as_tensor(np.ascontiguousarray(np.atleast_2d(targets), dtype=np.float32)
                             if not isinstance(targets, torch.Tensor) else targets).to(self.device, torch.float32)
        if tg.shape != (pos.shape[0], self.output_dim):
            raise ValueError(f"targets must be ({pos.shape[0]}, {self.output_dim}), got {tuple(tg.shape)}")
        mk = None
        if mask is not None:
            mk = torch.as_tensor(np.broadcast_to(np.asarray(mask, np.float32), tg.shape).copy()
                                 if not isinstance(mask, torch.Tensor) else mask).to(self.device, torch.float32)
        loss = self.train_step_device(pos, tg.contiguous(), None if mk is None else mk.contiguous())
        return float(loss.item())

    # ---- snapshots (VCSNAP1, cache.py:77-117) ---------------------------
    def save(self, path) -> None:
        arrays = self._param_dict()
        g = self.grid_cfg
        header = {
            "mode": self.mode, "output_dim": self.output_dim, "step": self.step,
            "grid": {**{k: v for k, v in asdict(g).items() if k not in ("aabb_min", "aabb_max")},
                     "aabb_min": g.aabb_min.tolist(), "aabb_max": g.aabb_max.tolist()},
            "train": asdict(self.train_cfg),
            "arrays": [{"name": k, "shape": list(v.shape)} for k, v in arrays.items()],
            "hidden_dims": list(self.net_cfg.hidden_dims),
        }
        blob = json.dumps(header).encode("utf-8")
        with open(path, "wb") as fh:
            fh.write(SNAP_MAGIC)
            fh.write(struct.pack("<I", len(blob)))
            fh.write(blob)
            for v in arrays.values():
                fh.write(np.ascontiguousarray(v, dtype="<f4").tobytes())

    @classmethod
    def load(cls, path, **kw) -> "VisibilityCache":
        with open(path, "rb") as fh:
            if fh.read(len(SNAP_MAGIC)) != SNAP_MAGIC:
                raise ValueError(f"{path}: not a cache snapshot")
            (hlen,) = struct.unpack("<I", fh.read(4))
            header = json.loads(fh.read(hlen).decode("utf-8"))
            hidden = tuple(header.get("hidden_dims", (32, 32)))
            obj = cls(mode=header["mode"], output_dim=header["output_dim"],
                      grid=HashGridConfig(**header["grid"]), train=TrainStepConfig(**header["train"]),
                      hidden_dims=hidden, **kw)
            obj.step = header["step"]
            arrays = obj._param_dict()
            for spec in header["arrays"]:
                shape = tuple(spec["shape"])
                arrays[spec["name"]][...] = np.frombuffer(fh.read(4 * int(np.prod(shape))),
                                                          dtype="<f4").reshape(shape)
        ws = [arrays[f"w{i}"] for i in range(len(obj.net_cfg.layer_dims))]
        bs = [arrays[f"b{i}"] for i in range(len(obj.net_cfg.layer_dims))]
        obj._upload(arrays["grid"], MLPParams(ws, bs))
        return obj


def make_cache(scene, mode: str, seed: int = 0, clusters: int | None = None,
               grid: HashGridConfig | None = None, train: TrainStepConfig | None = None,
               dtype=np.float32, **kw) -> VisibilityCache:
    """Cache sized to the scene: K lights, K clusters, or 3 RGB outputs (cache.py:120-139)."""
    box = {"aabb_min": scene.aabb_min, "aabb_max": scene.aabb_max}
    if mode == MODE_LIGHTS:
        out, grid = scene.n_lights, grid or HashGridConfig(**box)
    elif mode == MODE_CLUSTERS:
        if clusters is None:
            raise ValueError("cluster mode needs a cluster count")
        out, grid = clusters, grid or clustered_config(**box)
    elif mode == MODE_RADIANCE:
        out, grid = 3, grid or HashGridConfig(**box)
    else:
        raise ValueError(f"unknown cache mode {mode!r}")
    return VisibilityCache(mode, out, grid, train=train, seed=seed, dtype=dtype, **kw)
