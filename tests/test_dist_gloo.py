"""World-size-2 gloo tests of the multi-GPU logic on CPU.

The data-parallel train step is: every rank builds the same
global batch, computes gradients of its row shard [b*r/N, b*(r+1)/N) with
d_out scaled by the GLOBAL b*K, one allreduce (sum) of the fixed-point
gradient buffer + loss, then an identical Adam update on every rank.  Here the
per-rank gradient is the oracle's (CPU), quantised to the same 2^-48 fixed
point the CUDA scatter uses, so the test checks the exchange and the shard
arithmetic the GPU path relies on: the allreduced int64 gradient equals the
single-process full-batch one bit for bit, and ranks stay in lockstep.
Screen-tile sharding of the query needs no exchange; its global-draw-index
property is covered by tests/test_oracle.py::TestSampling::test_nls_sharded_matches_whole.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import vc_oracle as O

FX = 2.0 ** 48


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def shard_rows(b: int, r: int, n: int):
    return b * r // n, b * (r + 1) // n


def _setup():
    g = O.Grid(levels=4, features_per_level=2, table_size=1 << 10, aabb_min=(-1, 0, -1), aabb_max=(1, 1, 1))
    cache = O.Cache(g, 3, hidden=(16, 16), seed=2)
    rng = np.random.default_rng(7)
    pos = rng.uniform((-1, 0, -1), (1, 1, 1), (203, 3))
    tgt = (rng.random((203, 3)) < 0.5).astype(np.float32)
    return cache, pos, tgt


def _grad_fx_rows(cache, pos, tgt, lo, hi, b):
    """Per-contribution fixed point of one shard (what the CUDA scatter accumulates)."""
    feats, ctx = O.encode(cache.grid, cache.table, pos[lo:hi])
    out, zs, acts = O.mlp_forward(cache.ws, cache.bs, feats)
    _, _, d_in = O.mlp_backward(cache.ws, zs, acts, tgt[lo:hi], b_scale=b)
    gfx = np.zeros(cache.table.size, np.int64)
    for level, (idx, w) in enumerate(ctx):
        up = d_in[:, level * 2:(level + 1) * 2]
        contrib = (w[:, :, None] * up[:, None, :]).astype(np.float32).astype(np.float64)
        flat = (level * cache.grid.T + idx)[:, :, None] * 2 + np.arange(2)
        np.add.at(gfx, flat.reshape(-1), np.rint(contrib * FX).astype(np.int64).reshape(-1))
    loss_sum = float(np.sum((out - tgt[lo:hi]) ** 2) / out.shape[1])
    return gfx, loss_sum


def touched_entries(cache, pos):
    """Sorted table entries the whole (global) batch touches -- identical on every rank
    (restates nvc_exchange_index: 8 corners per (row, level), level-major entry ids)."""
    _, ctx = O.encode(cache.grid, cache.table, pos)
    ent = [level * cache.grid.T + idx.reshape(-1) for level, (idx, _) in enumerate(ctx)]
    return np.unique(np.concatenate(ent))


def _worker(rank, world, port, q, compact):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cache, pos, tgt = _setup()
    b = pos.shape[0]
    lo, hi = shard_rows(b, rank, world)
    gfx, ls = _grad_fx_rows(cache, pos, tgt, lo, hi, b)
    loss = torch.tensor([ls], dtype=torch.float64)
    if compact:   # GradExchange: allreduce only the entries the global batch touched
        ent = touched_entries(cache, pos)
        f = cache.grid.F
        cols = (ent[:, None] * f + np.arange(f)).reshape(-1)
        buf = torch.from_numpy(gfx[cols].copy())
        dist.all_reduce(buf)
        dist.all_reduce(loss)
        assert not np.delete(gfx, cols).any()        # untouched entries are zero on every rank
        gfx = np.zeros_like(gfx)
        gfx[cols] = buf.numpy()
        grad = torch.from_numpy(gfx)
    else:
        grad = torch.from_numpy(gfx)
        dist.all_reduce(grad)         # dense: sum of int64 fixed point
        dist.all_reduce(loss)
    g32 = (grad.numpy().astype(np.float64) / FX).astype(np.float32)
    p = cache.flat()
    st = O.Adam(p.size)
    full = np.zeros(p.size, np.float32)
    full[:g32.size] = g32
    st.step(p, full, O.lr_at(0))
    q.put((rank, grad.numpy(), float(loss.item()) / b, p))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,compact", [(2, False), (2, True)])
def test_dp_allreduce_matches_full_batch(world, compact):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, compact)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = sorted(q.get(timeout=120) for _ in range(world))
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    cache, pos, tgt = _setup()
    b = pos.shape[0]
    full_fx, full_loss = _grad_fx_rows(cache, pos, tgt, 0, b, b)
    for rank, gfx, loss, params in res:
        np.testing.assert_array_equal(gfx, full_fx)            # order-independent integer sum
        assert loss == pytest.approx(full_loss / b, rel=1e-6)   # f32 partial sums
    np.testing.assert_array_equal(res[0][3], res[1][3])      # ranks in lockstep after Adam
    # and the quantised gradient agrees with the reference-order FP32 scatter
    fx_f = full_fx.astype(np.float64) / FX
    loss_ref, g_ref = cache.grads(pos, tgt)
    np.testing.assert_allclose(fx_f, g_ref[:fx_f.size], rtol=1e-5, atol=1e-12)


def test_shard_rows_partition():
    for b in (0, 1, 7, 8192, 8193):
        for n in (1, 2, 3, 8):
            rows = [r for s in range(n) for r in range(*shard_rows(b, s, n))]
            assert rows == list(range(b))
