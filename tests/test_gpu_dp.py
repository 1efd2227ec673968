"""The data-parallel PRODUCT path with two processes.

Two ranks share cuda:0 and talk over gloo (CUDA tensors; NCCL refuses two
ranks on one device and this build has one GPU).  Each rank runs the real
``train_frame_device(shard=r, n_shards=2, comm=...)``: the same global batch
on both ranks, targets and gradients of its row shard with d_out scaled by the
global b*K, the compact GradExchange (index -> pack -> allreduce -> unpack)
and the Adam update -- replicated, or sharded (``set_optimizer_shard``: Adam
on half the table per rank, all-gather, fp16 table rebuild).  After three
frames both ranks' parameters and Adam moments (on the owned slices) must
equal a single-process full-batch run bit for bit (integer fixed-point
gradients, per 32-row block, make the sum independent of the split), and the
losses agree to 1e-12.
"""

import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

FRAMES = 3


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _make(seed=4):
    from paper_2506_05930_b200 import MODE_LIGHTS, HashGridConfig, VisibilityCache, scene_from_dict
    from paper_2506_05930_b200.scenes import boxes_scene
    scene = scene_from_dict(boxes_scene(8))
    grid = HashGridConfig(levels=8, table_size=1 << 14, features_per_level=2, aabb_min=scene.aabb_min,
                          aabb_max=scene.aabb_max)
    cache = VisibilityCache(MODE_LIGHTS, 8, grid, seed=seed, hidden_dims=(64, 64), device=torch.device("cuda", 0))
    return scene, cache


def _run(rank, world, port, sharded, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    from paper_2506_05930_b200 import TrainFrameConfig
    from paper_2506_05930_b200.training import train_frame_device
    dist.init_process_group("gloo", rank=rank, world_size=world)
    scene, cache = _make()
    cfg = TrainFrameConfig(n_world=1024, n_screen=1024, seed=4)

    def comm(buf, loss):                     # the sum-allreduce the exchange hands us
        dist.all_reduce(buf)
        dist.all_reduce(loss)

    def gather(buf):                         # the sharded optimizer's all-gather
        out = [torch.empty_like(buf) for _ in range(world)]
        dist.all_gather(out, buf)
        return torch.stack(out)

    if sharded:
        cache.set_optimizer_shard(rank, world, gather)
    losses = []
    for f in range(FRAMES):
        loss, _ = train_frame_device(scene, scene.camera, cache, cfg, frame=f, shard=rank, n_shards=world, comm=comm)
        losses.append(float(loss.item()))
    torch.cuda.synchronize()
    np.savez(os.path.join(out_dir, f"rank{rank}.npz"), params=cache.params.cpu().numpy(),
             m=cache.adam_m.cpu().numpy(), v=cache.adam_v.cpu().numpy(), table=cache.table_h.cpu().numpy(),
             losses=np.array(losses))
    dist.barrier()
    dist.destroy_process_group()


@pytest.fixture(scope="module")
def single():
    from paper_2506_05930_b200 import TrainFrameConfig
    from paper_2506_05930_b200.training import train_frame_device
    scene, cache = _make()
    cfg = TrainFrameConfig(n_world=1024, n_screen=1024, seed=4)
    losses = [float(train_frame_device(scene, scene.camera, cache, cfg, frame=f)[0].item()) for f in range(FRAMES)]
    return dict(params=cache.params.cpu().numpy(), m=cache.adam_m.cpu().numpy(), v=cache.adam_v.cpu().numpy(),
                table=cache.table_h.cpu().numpy(), losses=np.array(losses), grid=cache.grid_cfg.param_count,
                ranges=None)


@pytest.mark.parametrize("sharded", [False, True])
def test_two_rank_dp_equals_single_process(tmp_path, single, sharded):
    mp.start_processes(_run, args=(2, _free_port(), sharded, str(tmp_path)), nprocs=2, join=True,
                       start_method="spawn")
    for r in range(2):
        got = np.load(tmp_path / f"rank{r}.npz")
        np.testing.assert_array_equal(got["params"], single["params"])
        np.testing.assert_array_equal(got["table"], single["table"])
        # the loss is an f64 sum of per-block partials, split over the ranks
        np.testing.assert_allclose(got["losses"], single["losses"], rtol=1e-12)
        if not sharded:
            np.testing.assert_array_equal(got["m"], single["m"])
            np.testing.assert_array_equal(got["v"], single["v"])
    if sharded:      # each rank's Adam moments are current on the table slice it owns (+ the MLP)
        _, cache = _make()
        n = single["grid"]
        for r in range(2):
            got = np.load(tmp_path / f"rank{r}.npz")
            lo, hi = cache._adam_range(r, 2)
            for key in ("m", "v"):
                np.testing.assert_array_equal(got[key][lo:hi], single[key][lo:hi])
                np.testing.assert_array_equal(got[key][n:], single[key][n:])
