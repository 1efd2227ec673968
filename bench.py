"""Benchmark: one online NVC frame at 1080p x 32 lights (BASELINE.json configs[1]).

A step = one online frame, in the reference's order (render.py:297-324):
  1. training batch on the GPU: 4096 world + 4096 screen samples, 8192 x 32
     FP64 shadow-ray labels (training.py:166-199) -- generated one frame ahead
     on a side stream (it depends only on the frame index);
  2. one train step: encode -> MLP fwd/bwd -> fixed-point hash-grid scatter
     -> dense Adam over all 16.8 M parameters (cache.py:60-73);
  3. full-screen NLS query on the 1920x1080 G-buffer: hash-grid encode ->
     tcgen05 MLP 32-64-64-64-32 -> clamp * lum -> FP64 WRS with numpy Philox
     -> light point (sampling.py:184-205); the selection kernel runs on its
     own stream so it overlaps the next frame's train step.
Inputs (G-buffer, per-camera light-major lum table) are built once before
timing, as the reference memoizes them per camera (render.py:128-142).

`value` = visibility queries/s (all pixels, whole job) with inputs resident in
HBM; `e2e` = the same through the public device API with the G-buffer
positions copied H2D from pinned memory and (ids, points, W, loss) copied
back D2H every frame.  N > 1 (torchrun): weak scaling -- every rank renders its
own 1080p tile of an N-tile frame (global pixel ids keep the RNG draws
distinct) and trains data-parallel on its 8192-row shard of an 8192*N-row
global batch, with one NCCL allreduce of the fixed-point gradients per step.

`--impl reference` times the unmodified reference (baseline/_ref, installed by
tools/install_reference.sh) on the host cores with the same workload: its own
train_frame + nls_sample_batch on a 1/8 pixel sample (extrapolated); the CPU
oracle port (oracle/) stands in only when baseline/_ref is absent.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WIDTH, HEIGHT, K = 1920, 1080, 32
LEVELS, TABLE, FEATS, HIDDEN = 16, 1 << 19, 2, (64, 64, 64)
N_WORLD = N_SCREEN = 4096
# our kernels per online frame: batch (side stream) k_world, k_screen_round0,
# k_screen_finish, k_morton_order, k_targets_sorted; train k_tr_encode, k_train3,
# k_tr_scatter, k_reduce_parts, k_adam_bulk, k_adam_mlp; query k_enc_tiles2,
# k_mlp_ts, k_nls32g
LAUNCHES_PER_FRAME = 14
LUM_DEFAULT = "f64"
METRIC = "visibility queries/s (encode+MLP+WRS) at 1080p x 32 lights; train samples/s"
UNIT = "queries/s"
C4_METRIC = "visibility queries/s (encode+MLP+WRS) at 1080p x 128 lights (C4); train samples/s"
RENDER_METRIC = "rendered pixels/s (online frame: train + NLS + one shadow ray per pixel) at 1080p x 32 lights"


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None
        self.recording = True     # rows are kept only inside window() once it has been used
        self.seen = 0

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def settle(self, timeout: float = 3.0):
        """Wait for the first sample: nvidia-smi's start-up (a CPU burst) is over
        before a timed region begins, so it cannot delay the host's frame issue."""
        t0 = time.perf_counter()
        while self.proc is not None and self.seen == 0 and time.perf_counter() - t0 < timeout:
            time.sleep(0.02)
        self.recording = False
        self.rows = []

    class _Window:
        def __init__(self, s):
            self.s = s

        def __enter__(self):
            self.s.recording = True

        def __exit__(self, *exc):
            time.sleep(0.25)            # the sample covering the region's end
            self.s.recording = False

    def window(self):
        return ClockSampler._Window(self)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 6:
                self.seen += 1
                if self.recording:
                    self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.25)
            self.proc.terminate()
            self.proc.wait(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
# CPU side: the oracle port of the reference (cpu_baseline and --impl reference)
# ---------------------------------------------------------------------------

_CPU_STATE = {}   # (scene arrays, cache, G-buffer sample) inherited by forked workers


def _oracle_query_chunk(args):
    """Encode+MLP+WRS for a pixel chunk on one host core (oracle restatement)."""
    from oracle import vc_oracle as O
    lo, hi, key, p_first, p_total = args
    from threadpoolctl import threadpool_limits
    st = _CPU_STATE
    with threadpool_limits(1):       # one core per worker: no BLAS oversubscription
        vis = st["cache"].infer(st["pos"][lo:hi])
        return O.nls_sample(st["sa"], vis, st["lum"][lo:hi], key, p_total=p_total, p_first=p_first)


def cpu_reference(sample_pixels: int = 24576, procs: int | None = None, repeats: int = 1) -> dict:
    """Oracle port timed on the host: one full 8192-sample train step (batch
    generation + step) plus NLS on `sample_pixels` pixels of the 1080p frame;
    frame time extrapolates the query linearly to all pixels."""
    import multiprocessing as mp

    from oracle import vc_oracle as O
    from paper_2506_05930_b200.scene import scene_from_dict
    from paper_2506_05930_b200.scenes import boxes_scene

    procs = procs or os.cpu_count() or 1
    s = scene_from_dict(boxes_scene(32))
    cam = np.array([*s.camera.position, *s.camera.look_at, *s.camera.up, s.camera.fov_deg, WIDTH, HEIGHT], float)
    sa = O.SceneArrays(s.triangles_v0, s.triangles_v1, s.triangles_v2, s.tri_material, s.tri_light, s.lt_kind,
                       s.lt_verts, s.lt_normal, s.lt_radiance, s.mat_albedo, cam)
    grid = O.Grid(levels=LEVELS, features_per_level=FEATS, table_size=TABLE, aabb_min=s.aabb_min,
                  aabb_max=s.aabb_max)
    cache = O.Cache(grid, K, hidden=HIDDEN, seed=0)
    # G-buffer sample: evenly strided pixels of the 1080p frame (memoized per camera, untimed)
    p_total = WIDTH * HEIGHT
    pix = np.linspace(0, p_total - 1, sample_pixels).astype(np.int64)
    jit = O.uniform_at(O.stream_key("primary"), np.stack([2 * pix, 2 * pix + 1], 1))
    ys, xs = np.divmod(pix, WIDTH)
    o, d = sa.camera_rays(xs + jit[:, 0], ys + jit[:, 1])
    gb = sa.trace(o, d)
    lum = sa.lum(sa.factors(gb["position"], gb["normal"]), gb["albedo"])
    key = O.stream_key(0, 0, "light-select")
    best_train, best_query = float("inf"), float("inf")
    bounds = [(int(c[0]), int(c[-1]) + 1) for c in np.array_split(np.arange(sample_pixels), procs) if c.size]
    ctx = mp.get_context("fork")
    for rep in range(repeats):
        t0 = time.perf_counter()
        pos, tgt = O.train_batch(sa, 0, rep)
        cache.train_step(pos, tgt)
        t1 = time.perf_counter()
        # workers fork after the step and inherit the trained cache (no pickling of 16.8 M parameters)
        _CPU_STATE.update(sa=sa, cache=cache, pos=gb["position"], lum=lum)
        with ctx.Pool(procs) as pool:
            pool.map(_oracle_query_chunk, [(lo, lo + 1, key, lo, p_total) for lo, _ in bounds])   # warm-up
            t2 = time.perf_counter()
            pool.map(_oracle_query_chunk, [(lo, hi, key, lo, p_total) for lo, hi in bounds])
            t3 = time.perf_counter()
        best_train, best_query = min(best_train, t1 - t0), min(best_query, t3 - t2)
    frame_s = best_train + best_query * (p_total / sample_pixels)
    return {"value": p_total / frame_s, "unit": UNIT, "cores": procs, "kind": "port",
            "sample": (f"oracle port (numpy + serial C geometry) on host: 1 full train step "
                       f"(8192 samples, {best_train:.2f} s, 1 process) + NLS on {sample_pixels} strided "
                       f"pixels of the 1080p frame ({best_query:.2f} s over {procs} processes), query "
                       f"extrapolated x{p_total / sample_pixels:.1f}; frame {frame_s:.1f} s"),
            "train_samples_per_s": (N_WORLD + N_SCREEN) / frame_s, "frame_s": frame_s}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def gpu_arm(args) -> None:
    import torch
    import torch.distributed as dist

    from paper_2506_05930_b200 import MODE_LIGHTS, HashGridConfig, TrainFrameConfig, VisibilityCache
    from paper_2506_05930_b200 import _lib
    from paper_2506_05930_b200 import rng as R
    from paper_2506_05930_b200.render import gbuffer_device, shade_device
    from paper_2506_05930_b200.sampling import PixelCtx, nls_sample_device
    from paper_2506_05930_b200.scene import scene_from_dict
    from paper_2506_05930_b200.scenes import boxes_scene, rooms_scene
    from paper_2506_05930_b200.training import BatchPipeline, train_frame_device

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # NVC_RANKS_PER_GPU=n (test only): n ranks share a GPU over gloo -- the N>1
    # code path on a 1-GPU box (no kernel waits on another rank; NCCL refuses it)
    local = int(os.environ.get("LOCAL_RANK", "0")) // int(os.environ.get("NVC_RANKS_PER_GPU", "1"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    prio = int(os.environ.get("NVC_MAIN_PRIORITY", "-1"))
    if prio:
        torch.cuda.set_stream(torch.cuda.Stream(dev, priority=prio))
    if world > 1:
        if os.environ.get("NVC_RANKS_PER_GPU"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)

    c4 = args.workload == "c4"
    kk, hid = (128, (128, 128, 128)) if c4 else (K, HIDDEN)
    scene = scene_from_dict(rooms_scene(128) if c4 else boxes_scene(32))
    cam = scene.camera.resized(WIDTH, HEIGHT * world)      # N tiles of 1080 rows
    P = WIDTH * HEIGHT
    p_first, p_total = rank * P, P * world
    pos, nrm, alb, hit, _ = gbuffer_device(scene, cam, p_first, P)
    # luminance table precision: NVC_LUM=f64 (the reference's) or f32 (default perf path:
    # half the NLS table traffic; its light-choice mismatch vs f64 is measured in
    # tests/test_gpu_headline.py::test_c2_f32_lum_choice_mismatch)
    lum_dt = np.float64 if os.environ.get("NVC_LUM", LUM_DEFAULT) == "f64" else np.float32
    ctx = PixelCtx(scene, pos, nrm, alb, table_dtype=lum_dt)
    ctx.lum_device()
    grid = HashGridConfig(levels=LEVELS, table_size=TABLE, features_per_level=FEATS, aabb_min=scene.aabb_min,
                          aabb_max=scene.aabb_max)
    cache = VisibilityCache(MODE_LIGHTS, kk, grid, seed=0, hidden_dims=hid, device=dev)
    if os.environ.get("NVC_COMPACT"):    # compact gradient slots (the DP exchange layout) also at N=1
        cache.set_compact(True)
    if os.environ.get("NVC_L2_PIN"):      # measured slower (it starves the streaming Adam of L2)
        cache.pin_table_in_l2()
    # one training step per frame on the reference's batch (4096 world + 4096 screen
    # samples of the N-tile frame), its rows sharded over the ranks: the gradient
    # exchange (the batch's touched entries) stays ~17 MB at any N
    cfg = TrainFrameConfig(n_world=N_WORLD, n_screen=N_SCREEN, seed=0)
    # training batches are generated one frame ahead on a side stream (they depend on
    # the frame index only), overlapping the FP64 ray kernels with training + query
    pipe = BatchPipeline(scene, cam, cfg, kk, dev, rank, world, cache=cache)
    out = (torch.empty(P, dtype=torch.int64, device=dev), torch.empty((P, 3), dtype=torch.float64, device=dev),
           torch.empty(P, dtype=torch.float64, device=dev))

    def comm(grad_fx, loss):
        dist.all_reduce(grad_fx)
        dist.all_reduce(loss)

    if world > 1 and os.environ.get("NVC_SHARD_OPT"):
        # sharded optimizer: Adam on 1/N of the table per rank + an
        # all-gather of the updated slices (off by default: at C2 the 67 MB
        # all-gather costs more than the replicated 121 us Adam it replaces)
        def gather(buf):
            if dist.get_backend() == "gloo":    # the NVC_RANKS_PER_GPU test mode
                parts = [torch.empty_like(buf) for _ in range(world)]
                dist.all_gather(parts, buf)
                return torch.stack(parts)
            out = torch.empty((world, buf.numel()), dtype=buf.dtype, device=buf.device)
            dist.all_gather_into_tensor(out, buf)
            return out
        cache.set_optimizer_shard(rank, world, gather)

    stream = torch.cuda.current_stream()
    marks = [torch.cuda.Event(enable_timing=True) for _ in range(4)]

    last_bufs = [None]

    # the NLS selection of frame f runs on its own stream, overlapping frame f+1's
    # train step (it reads only the visibilities, luminances and scene)
    sel_stream = (torch.cuda.Stream(dev, priority=int(os.environ.get("NVC_SELECT_PRIORITY", "0")))
                  if not os.environ.get("NVC_SELECT_INLINE") else None)

    shade = args.workload == "render"
    rgb_buf = [torch.empty((P, 3), dtype=torch.float64, device=dev) for _ in range(2)] if shade else [None, None]

    # NVC_DIAG=no-train / no-query / no-nls (diagnostics only, never a bench value):
    # drop part of the frame to see which work bounds the overlapped frame
    diag = os.environ.get("NVC_DIAG", "")

    def frame_into(f, outs, timed_parts=None, rgb=None):
        if timed_parts is not None:
            marks[0].record(stream)
        if diag != "no-train" or f < args.warmup:
            loss, bufs = train_frame_device(scene, cam, cache, cfg, frame=f, shard=rank, n_shards=world,
                                            comm=comm if world > 1 else None, pipeline=pipe)
            last_bufs[0] = bufs
        else:
            loss = last_bufs[0].loss[1]
        if timed_parts is not None:
            marks[1].record(stream)
        if diag == "no-nls":       # encoder + MLP only (what a free NLS would leave)
            ws = cache.query_workspace(P)
            _lib.call("nvc_query_front", cache.model, ctx.pos.data_ptr(), P, _lib.ptr(ws), _lib.stream_ptr())
        elif diag != "no-query":
            nls_sample_device(ctx, cache, R.stream_key(0, f, "light-select"), 0, p_first=p_first, p_total=p_total,
                              out=outs, select_stream=None if timed_parts is not None else sel_stream)
        if timed_parts is not None:
            marks[2].record(stream)
        if shade:   # pass 5: one shadow ray per pixel to its NLS-selected light point
            if timed_parts is None and sel_stream is not None:
                with torch.cuda.stream(sel_stream):
                    shade_device(scene, ctx.pos, ctx.nrm, ctx.alb, *outs, out=rgb)
                    done = torch.cuda.Event()
                    done.record(sel_stream)
                    cache.select_done = done
            else:
                shade_device(scene, ctx.pos, ctx.nrm, ctx.alb, *outs, out=rgb)
            if timed_parts is not None:
                marks[3].record(stream)
        return loss

    def frame(f, timed_parts=None):
        return frame_into(f, out, timed_parts, rgb_buf[0])

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up (also validates the batch never shrinks) ----
    for f in range(args.warmup):
        frame(f)
    barrier()
    assert int(last_bufs[0].n_rows.item()) == cfg.n_world + cfg.n_screen, "screen rays missed: batch shrank"

    if os.environ.get("NVC_TIMELINE"):   # diagnostics: a CUPTI kernel timeline of 12 frames (tools/timeline.py)
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for f in range(12):
                frame(args.warmup + f)
            if cache.select_done is not None:
                stream.wait_event(cache.select_done)
            barrier()
        prof.export_chrome_trace(os.environ["NVC_TIMELINE"])
        return

    # the clock sampler starts now (its start-up must not overlap the timed region)
    sampler = ClockSampler(local).__enter__()
    # ---- per-stage split (separate pass, events between stages and between
    #      the three query kernels, all on the launching stream); frame numbers
    #      continue the sequence so the batch pipeline's prefetch stays valid ----
    split_train, split_query, split_k, split_shade = [], [], [], []
    kms = (ctypes.c_float * 3)()
    n_split = min(args.steps, 10)
    for f in range(n_split):
        _lib.call("nvc_profile_stages", 1)
        frame(args.warmup + f, timed_parts=True)
        _lib.call("nvc_profile_stages", 0)
        marks[3 if shade else 2].synchronize()
        if diag not in ("no-query", "no-nls"):
            _lib.call("nvc_profile_stage_ms", ctypes.addressof(kms))
        if shade:
            split_shade.append(marks[2].elapsed_time(marks[3]))
        split_train.append(marks[0].elapsed_time(marks[1]))
        split_query.append(marks[1].elapsed_time(marks[2]))
        split_k.append(list(kms))

    # ---- timed region: K frames, inputs resident ----
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    f0 = args.warmup + n_split        # its batch was prefetched by the last split frame
    sampler.settle()
    barrier()
    with sampler as clocks, clocks.window():
        if os.environ.get("NVC_PREQUEUE"):   # diagnostic: let the host run ahead of the GPU
            torch.cuda._sleep(int(os.environ["NVC_PREQUEUE"]))
        start.record(stream)
        t_issue = time.perf_counter()
        for f in range(args.steps):
            loss = frame(f0 + f)
        if cache.select_done is not None:
            stream.wait_event(cache.select_done)
        end.record(stream)
        issue_ms = (time.perf_counter() - t_issue) * 1e3 / args.steps   # host time to enqueue a frame
        barrier()
    ms = start.elapsed_time(end) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    if diag:                          # diagnostics: the frame time only, never a bench line
        if rank == 0:
            print(json.dumps({"diag": diag, "ms_per_step": ms, "steps": args.steps}), flush=True)
        return

    # ---- e2e: host G-buffer positions in, (ids, points, W, loss) out, every frame ----
    # Copies run on their own streams (H2D and D2H engines) double-buffered
    # against the compute stream: frame f+1's positions upload and frame f-1's
    # results download while frame f computes.
    pos_host = pos.cpu().pin_memory()
    outs_host = [torch.empty(o.shape, dtype=o.dtype, pin_memory=True) for o in ((rgb_buf[0],) if shade else out)]
    loss_host = torch.empty(1, dtype=torch.float64, pin_memory=True)
    pos_buf = [ctx.pos, torch.empty_like(ctx.pos)]
    out_buf = [out, tuple(torch.empty_like(o) for o in out)]
    s_h2d, s_d2h = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    ev_h2d = [torch.cuda.Event() for _ in range(2)]
    ev_comp = [torch.cuda.Event() for _ in range(2)]
    ev_d2h = [torch.cuda.Event() for _ in range(2)]
    for e in ev_comp + ev_d2h:
        e.record(stream)
    e2e_steps = max(3, min(args.steps, 20))
    barrier()
    start.record(stream)
    for f in range(e2e_steps):
        b = f % 2
        with torch.cuda.stream(s_h2d):
            s_h2d.wait_event(ev_comp[b])              # frame f-2's main-stream kernels are done with it
            s_h2d.wait_event(ev_d2h[b])               # ... and its select-stream work (render: shading reads pos)
            pos_buf[b].copy_(pos_host, non_blocking=True)
            ev_h2d[b].record(s_h2d)
        stream.wait_event(ev_h2d[b])
        stream.wait_event(ev_d2h[b])                  # frame f-2's results are downloaded
        if sel_stream is not None:
            sel_stream.wait_event(ev_d2h[b])
        ctx.pos = pos_buf[b]
        loss = frame_into(f0 + args.steps + f, out_buf[b], rgb=rgb_buf[b])
        ev_comp[b].record(stream)
        with torch.cuda.stream(s_d2h):
            s_d2h.wait_event(ev_comp[b])
            if cache.select_done is not None:
                s_d2h.wait_event(cache.select_done)
            for h, d in zip(outs_host, (rgb_buf[b],) if shade else out_buf[b]):
                h.copy_(d, non_blocking=True)
            loss_host.copy_(loss.reshape(1), non_blocking=True)
            ev_d2h[b].record(s_d2h)
    for e in ev_d2h:
        stream.wait_event(e)
    if cache.select_done is not None:
        stream.wait_event(cache.select_done)
    end.record(stream)
    barrier()
    ctx.pos = pos_buf[0]
    e2e_ms = start.elapsed_time(end) / e2e_steps
    t = torch.tensor([e2e_ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    e2e_ms = float(t.item())

    if rank == 0:
        hbm, tflops, src = peaks()
        q_ms = statistics.median(split_query)
        tr_ms = statistics.median(split_train)
        k_ms = [statistics.median(x[i] for x in split_k) for i in range(3)]
        # roofline of each query kernel: algorithmic work per launch / its event-timed duration
        # (DESIGN.md section 4 gives the per-pixel figures)
        lum_b = np.dtype(lum_dt).itemsize
        lum_nnz = int(torch.count_nonzero(ctx.lum_device()).item())
        dims = (LEVELS * FEATS,) + tuple(hid) + (kk,)
        flop_px = 2 * sum(a * b for a, b in zip(dims[:-1], dims[1:]))
        kern = {
            "k_enc_tiles2": ("hbm", P * (24 + 64), k_ms[0]),             # pos in, fp16 feature tile out
            "k_mlp_ts": ("tensor", P * flop_px, k_ms[1]),                # 24,576 flop per pixel
            # vis row + mask in, id/W/point out per pixel, plus the luminances of the
            # nonzero (pixel, light) pairs only: zero-weight lights are never read
            "k_nls32": ("hbm", P * (2 * kk + 4 * ((kk + 31) // 32) + 40) + lum_b * lum_nnz, k_ms[2]),
        }
        # roofline denominators measured on this GPU in this run (tools/rooflines.py,
        # libnvc_micro.so): Philox block rate, L2 streaming read, random L2 gathers
        try:
            sys.path.insert(0, os.path.join(ROOT, "tools"))
            import rooflines
            roof = rooflines.measure(quick=True)
        except Exception as exc:      # microbenchmarks absent: report without them
            roof = {"error": str(exc)[:200]}
        enc_gathers = P * LEVELS * 4 / (k_ms[0] * 1e-3) / 1e9
        probe = roof.get("l2_gather_G_per_s_67MB")
        l2_peak = max((v for k, v in roof.items() if k.startswith("l2_stream_GBps")), default=None)
        # NLS Philox work: one block per nonzero 4-light group + the light-point pair
        m = ctx.mask_device("lum").view(torch.int32)
        groups = sum(((m >> (4 * g)) & 15).ne(0).sum().item() for g in range(8)) if kk <= 32 else None
        nls_blocks = (groups + P) if groups is not None else None
        # headline kernel: the NLS -- it closes every frame (select stream, resident
        # ~340 of the ~585 us per frame beside the training half, profiles/r2_timeline_c2.txt);
        # the encoder's time alone is within 1 % of it, but the encoder is bound by L2
        # gathers (its L2 roofline is roofline.encoder_l2), so ranking by isolated time
        # would flip between the two from run to run
        name = "k_nls32" if "k_nls32" in kern else max(kern, key=lambda k: kern[k][2])
        bound, work, kms = kern[name]
        if bound == "tensor":
            achieved, peak, unit = work / (kms * 1e-3) / 1e12, tflops, "TFLOP/s"
        else:
            achieved, peak, unit = work / (kms * 1e-3) / 1e9, hbm, "GB/s"
        traffic = None
        prof = os.path.join(ROOT, "profiles", "kernel_dram_bytes.json")
        if os.path.exists(prof):
            try:   # ncu dram__bytes_read+write per launch of that kernel (profiles/, committed)
                traffic = next((v for k, v in json.load(open(prof)).items() if k.startswith(name)), None)
            except Exception:
                traffic = None
        clk = clocks.summary()
        metric, munit = (RENDER_METRIC, "pixels/s") if shade else ((C4_METRIC, UNIT) if c4 else (METRIC, UNIT))
        line = {
            "metric": metric, "value": P * world / (ms * 1e-3), "unit": munit, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "fp16 MLP / fp64 index+WRS / fp32 train",
            "data": f"synthetic ({'rooms_scene(128)' if c4 else 'boxes_scene(32)'} fixture, random-init weights, seed 0)",
            "config": {"workload": (f"C4: {WIDTH}x{HEIGHT * world} rooms128 (K=128), L=16 T=2^19 F=2, MLP 3x128, "
                                    if c4 else
                                    f"C2: {WIDTH}x{HEIGHT * world} boxes32 (K=32), L=16 T=2^19 F=2, MLP 3x64, ")
                                   + f"1 online frame = train batch {N_WORLD + N_SCREEN} (rows sharded over {world} ranks) "
                                   + "+ NLS over all pixels"
                                   + (" + one shadow ray per pixel (shade_batch)" if shade else ""),
                       "train_samples_per_s": (N_WORLD + N_SCREEN) / (ms * 1e-3),
                       "pixels_per_gpu": P, "global_batch": N_WORLD + N_SCREEN,
                       "parallelism": f"dp{world} (train: batch rows sharded, one allreduce) + {world} screen tiles (query)",
                       "l2": (f"inputs > L2 every frame (lum table {P * kk * lum_b / 1e6:.0f} MB "
                              f"{np.dtype(lum_dt).name} + 16.8 M-parameter Adam stream 530 MB)"),
                       "lum_dtype": np.dtype(lum_dt).name,
                       "lum_nonzero_per_pixel": lum_nnz / P,
                       "host_issue_ms_per_frame": issue_ms,
                       "stage_ms": {"train_frame": tr_ms, "query": q_ms, "k_enc_tiles2": k_ms[0],
                                    "k_mlp_ts": k_ms[1], "k_nls32": k_ms[2],
                                    **({"k_shade": statistics.median(split_shade)} if shade else {})}},
            "e2e": {"value": P * world / (e2e_ms * 1e-3), "unit": munit,
                    "h2d_bytes_per_step": int(pos_host.numel() * 8),
                    "d2h_bytes_per_step": int(sum(h.numel() * h.element_size() for h in outs_host) + 8)},
            "gpu_launches": (LAUNCHES_PER_FRAME + int(shade)) * args.steps,
            "roofline": {"bound": bound, "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak,
                         "traffic": traffic, "kernel": name, "peak_source": src,
                         "work_per_launch": work, "launch_ms": kms,
                         "all": {k: {"bound": v[0], "ms": v[2],
                                     "frac": (v[1] / (v[2] * 1e-3) / (1e12 * tflops if v[0] == "tensor" else 1e9 * hbm))}
                                 for k, v in kern.items()},
                         "encoder_l2": {"gathers_G_per_s": enc_gathers, "payload_GBps": enc_gathers * 8,
                                        "l2_stream_peak_GBps": l2_peak,
                                        "frac_of_l2_stream": (enc_gathers * 8 / l2_peak) if l2_peak else None,
                                        "random_gather_probe_G_per_s": probe,
                                        "vs_random_probe": (enc_gathers / probe) if probe else None},
                         "nls_issue": ({"bound": "philox", "blocks_per_launch": nls_blocks,
                                        "achieved_blocks_per_s": nls_blocks / (k_ms[2] * 1e-3),
                                        "peak_blocks_per_s": roof["philox_blocks_per_s"],
                                        "frac": nls_blocks / (k_ms[2] * 1e-3) / roof["philox_blocks_per_s"]}
                                       if nls_blocks and "philox_blocks_per_s" in roof else None),
                         "microbench": roof},
            "clocks": clk,
        }
        assert line["roofline"]["unit"] in ("GB/s", "TFLOP/s") and line["roofline"]["bound"] in ("hbm", "tensor")
        if world == 1 and not args.no_cpu_baseline and not shade and not c4:
            line["cpu_baseline"] = cpu_baseline()
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def ndi4k_arm(args) -> None:
    """C3 (BASELINE.json configs[2]): Neural DI at 3840x2160 x 32 lights, screen-tile
    sharded (rank r renders rows [r*H/N, (r+1)*H/N) of the frame, no communication).
    One step = encoder + tcgen05 MLP + the FP64 Neural-DI sum over all of the
    rank's pixels with the G-buffer and per-camera factor table resident."""
    import torch
    import torch.distributed as dist

    from paper_2506_05930_b200 import MODE_LIGHTS, HashGridConfig, VisibilityCache
    from paper_2506_05930_b200.render import gbuffer_device
    from paper_2506_05930_b200.sampling import PixelCtx, neural_di_device
    from paper_2506_05930_b200.scene import scene_from_dict
    from paper_2506_05930_b200.scenes import boxes_scene

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    # NVC_RANKS_PER_GPU=n (test only): n ranks share a GPU over gloo -- the N>1
    # code path on a 1-GPU box (no kernel waits on another rank; NCCL refuses it)
    local = int(os.environ.get("LOCAL_RANK", "0")) // int(os.environ.get("NVC_RANKS_PER_GPU", "1"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if os.environ.get("NVC_RANKS_PER_GPU"):
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    W4, H4 = 3840, 2160
    scene = scene_from_dict(boxes_scene(32))
    cam = scene.camera.resized(W4, H4)
    rows = H4 // world
    P = W4 * rows
    pos, nrm, alb, _, _ = gbuffer_device(scene, cam, rank * P, P)
    ctx = PixelCtx(scene, pos, nrm, alb, table_dtype=np.float32)
    ctx.factor_device()
    ctx.mask_device("factor")
    grid = HashGridConfig(levels=LEVELS, table_size=TABLE, features_per_level=FEATS, aabb_min=scene.aabb_min,
                          aabb_max=scene.aabb_max)
    cache = VisibilityCache(MODE_LIGHTS, K, grid, seed=0, hidden_dims=HIDDEN, device=dev)
    out = torch.empty((P, 3), dtype=torch.float64, device=dev)
    for _ in range(args.warmup):
        neural_di_device(ctx, cache, out=out)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        s.record()
        for _ in range(args.steps):
            neural_di_device(ctx, cache, out=out)
        e.record()
        torch.cuda.synchronize()
    ms = s.elapsed_time(e) / args.steps
    t = torch.tensor([ms], device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dist.barrier()
    ms = float(t.item())
    if rank == 0:
        print(json.dumps({"metric": "neural DI queries/s at 3840x2160 x 32 lights (encode+MLP+NDI)",
                          "value": P * world / (ms * 1e-3), "unit": "queries/s", "n_gpus": world,
                          "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
                          "scaling": "strong", "vs_baseline": None, "dtype": "fp16 MLP / fp64 NDI sum",
                          "data": "synthetic (boxes_scene(32) fixture, random-init weights, seed 0)",
                          "config": {"workload": f"C3: {W4}x{H4} boxes32 (K=32) Neural DI, {world} screen tiles",
                                     "pixels_per_gpu": P},
                          "gpu_launches": 3 * args.steps, "clocks": clocks.summary()}), flush=True)
    if world > 1:
        dist.destroy_process_group()


def sweep_arm(args) -> None:
    """C5: query throughput sweep, N = 2^16 .. 2^26 shading points x
    K in {8, 32, 128} (boxes8 / boxes32 / rooms128).  Points ~ U(scene AABB) from
    the reference stream ("sweep"), normals +y, albedo 0.73; one step = encoder +
    tcgen05 MLP + FP64 WRS + light point over all N points (inputs resident).
    Grid L=16 T=2^19 F=2; MLP 3x64 for K <= 32, 3x128 for K = 128 (C4)."""
    import torch

    from paper_2506_05930_b200 import MODE_LIGHTS, HashGridConfig, VisibilityCache
    from paper_2506_05930_b200 import rng as R
    from paper_2506_05930_b200.sampling import PixelCtx, nls_sample_device
    from paper_2506_05930_b200.scene import scene_from_dict
    from paper_2506_05930_b200.scenes import boxes_scene, rooms_scene

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    max_log2 = int(os.environ.get("NVC_SWEEP_MAX_LOG2", "26"))
    rows = []
    for k, mk, hid in ((8, lambda: boxes_scene(8), (64, 64, 64)), (32, lambda: boxes_scene(32), (64, 64, 64)),
                       (128, lambda: rooms_scene(128), (128, 128, 128))):
        scene = scene_from_dict(mk())
        n_max = 1 << max_log2
        g = R.stream(0, "sweep")
        pos_all = torch.from_numpy(g.uniform(scene.aabb_min, scene.aabb_max, (n_max, 3))).to(dev)
        grid = HashGridConfig(levels=LEVELS, table_size=TABLE, features_per_level=FEATS, aabb_min=scene.aabb_min,
                              aabb_max=scene.aabb_max)
        cache = VisibilityCache(MODE_LIGHTS, k, grid, seed=0, hidden_dims=hid, device=dev)
        for lg in range(16, max_log2 + 1, 2):
            n = 1 << lg
            pos = pos_all[:n]
            nrm = torch.zeros_like(pos)
            nrm[:, 1] = 1.0
            alb = torch.full_like(pos, 0.73)
            ctx = PixelCtx(scene, pos, nrm, alb, table_dtype=np.float32)
            ctx.lum_device()
            ctx.mask_device("lum")
            key = R.stream_key(0, lg, "light-select")
            for _ in range(args.warmup):
                nls_sample_device(ctx, cache, key)
            reps = max(2, min(args.steps, int(2e8 // (n * max(k, 32)))))
            st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            st.record()
            for _ in range(reps):
                nls_sample_device(ctx, cache, key)
            en.record()
            torch.cuda.synchronize()
            ms = st.elapsed_time(en) / reps
            rows.append({"n": n, "k": k, "ms": ms, "queries_per_s": n / (ms * 1e-3), "reps": reps})
            del ctx, nrm, alb
            torch.cuda.empty_cache()
        del cache, pos_all
        torch.cuda.empty_cache()
    head = max((r for r in rows if r["k"] == 32), key=lambda r: r["n"])
    print(json.dumps({"metric": "visibility queries/s (encode+MLP+WRS), C5 sweep; value at the largest N, K=32",
                      "value": head["queries_per_s"], "unit": "queries/s", "n_gpus": 1, "steps": head["reps"],
                      "warmup": args.warmup, "ms_per_step": head["ms"], "higher_is_better": True, "scaling": "weak",
                      "vs_baseline": None, "dtype": "fp16 MLP / fp64 index+WRS",
                      "data": "synthetic (points U(AABB) from stream (0, 'sweep'), normals +y, albedo 0.73)",
                      "config": {"workload": "C5: N = 2^16..2^%d x K in {8 (boxes8), 32 (boxes32), 128 (rooms128)}"
                                             % max_log2, "sweep": rows}}), flush=True)


def clusters_arm(args) -> None:
    """Clustered NVC: rooms_scene(1024) (1024 lights) in 32
    k-means clusters at 1920x1080; one step = a cluster-mode train step on the
    C-config batch (24,576 world + 24,576 screen samples, cluster targets) + the
    two-step clustered light selection over all pixels (inputs resident)."""
    import torch

    from paper_2506_05930_b200 import TrainFrameConfig, make_cache
    from paper_2506_05930_b200 import rng as R
    from paper_2506_05930_b200.clusters import kmeans_cluster
    from paper_2506_05930_b200.render import gbuffer_device
    from paper_2506_05930_b200.sampling import PixelCtx, clustered_sample_device
    from paper_2506_05930_b200.scene import scene_from_dict
    from paper_2506_05930_b200.scenes import rooms_scene
    from paper_2506_05930_b200.training import BatchPipeline, train_frame_device

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", "0")))
    torch.cuda.set_device(dev)
    prio = int(os.environ.get("NVC_MAIN_PRIORITY", "-1"))   # as gpu_arm: the batch stream (-2) outranks the frame
    if prio:
        torch.cuda.set_stream(torch.cuda.Stream(dev, priority=prio))
    scene = scene_from_dict(rooms_scene(1024))
    cs = kmeans_cluster(scene.lights, 32, R.stream(0, R.CLUSTERING))
    cam = scene.camera.resized(WIDTH, HEIGHT)
    P = WIDTH * HEIGHT
    pos, nrm, alb, _, _ = gbuffer_device(scene, cam, 0, P)
    ctx = PixelCtx(scene, pos, nrm, alb, table_dtype=np.float64)   # per-camera f64 factor table (memoized)
    ctx.factor_device()
    cache = make_cache(scene, "clusters", seed=0, clusters=cs.m, device=dev)
    cfg = TrainFrameConfig.clustered()
    pipe = BatchPipeline(scene, cam, cfg, cs.m, dev, cache=cache, clusters=cs)
    split = {"train": [], "select": []}
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]

    def frame(f, timed=False):
        if timed:
            ev[0].record()
        train_frame_device(scene, cam, cache, cfg, frame=f, pipeline=pipe, clusters=cs)
        if timed:
            ev[1].record()
        clustered_sample_device(ctx, cache, cs, R.stream_key(0, f, R.LIGHT_SELECT))
        if timed:
            ev[2].record()

    for f in range(args.warmup):
        frame(f)
    for f in range(3):
        frame(100 + f, timed=True)
        torch.cuda.synchronize()
        split["train"].append(ev[0].elapsed_time(ev[1]))
        split["select"].append(ev[1].elapsed_time(ev[2]))
    steps = min(args.steps, 50)
    st, en = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    with ClockSampler(dev.index or 0) as clocks:
        st.record()
        for f in range(steps):
            frame(args.warmup + f)
        en.record()
        torch.cuda.synchronize()
    ms = st.elapsed_time(en) / steps
    print(json.dumps({"metric": "clustered-NVC frames: light selections/s at 1080p x 1024 lights in 32 clusters "
                                "(train step + two-step selection)",
                      "value": P / (ms * 1e-3), "unit": "queries/s", "n_gpus": 1, "steps": steps,
                      "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
                      "vs_baseline": None, "dtype": "fp16 MLP / fp64 factors+WRS / fp32 train",
                      "data": "synthetic (rooms_scene(1024), 32 k-means clusters, random-init weights, seed 0)",
                      "config": {"workload": f"clustered NVC: {WIDTH}x{HEIGHT} rooms1024 (K=1024, m=32 clusters), "
                                             f"train batch {cfg.n_world + cfg.n_screen}",
                                 "stage_ms": {k: statistics.median(v) for k, v in split.items()}},
                      "clocks": clocks.summary()}), flush=True)


REF_DIR = os.path.join(ROOT, "baseline", "_ref")
_REF_STATE = {}   # reference scene / cache / G-buffer sample, inherited by forked workers


def _import_reference():
    """The unmodified reference package installed into baseline/_ref (DESIGN 6), or None."""
    if not os.path.isdir(os.path.join(REF_DIR, "viscache")):
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nvc_numba_cache")
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    try:
        import viscache  # noqa: F401
        return viscache
    except Exception:
        return None


def _ref_nls_shard(args):
    """Reference nls_sample_batch on one contiguous shard of the pixel sample
    (one worker process, BLAS pinned to one thread)."""
    from threadpoolctl import threadpool_limits
    from viscache import rng as RR
    from viscache.sampling import PixelCtx as RefCtx, nls_sample_batch as ref_nls
    lo, hi, frame = args
    st = _REF_STATE
    ctxs = st.setdefault("ctxs", {})
    with threadpool_limits(1):
        if (lo, hi) not in ctxs:       # per-camera memo, as render.py:128-142 keeps it
            ctxs[(lo, hi)] = RefCtx(st["scene"], st["pos"][lo:hi], st["nrm"][lo:hi], st["alb"][lo:hi])
        t0 = time.perf_counter()
        ref_nls(ctxs[(lo, hi)], st["cache"], RR.stream(0, frame, "light-select"))
        return time.perf_counter() - t0


def reference_cpu(steps: int = 3, warmup: int = 1, every: int = 8, procs: int | None = None) -> dict:
    """The unmodified reference (baseline/_ref) timed on the host cores.

    One step = the reference's own ``train_frame`` (full 8192-sample batch,
    shadow-ray labels, train step; one process, as the reference runs) + its
    ``nls_sample_batch`` over every ``every``-th pixel of the 1080p G-buffer,
    split into contiguous shards over ``procs`` worker processes (BLAS pinned
    to one thread each; a harness around the reference's function, not a
    change to it).  The frame time extrapolates the query x``every``.  The
    G-buffer and per-camera luminance tables are built before timing (the
    reference memoizes them per camera).  Workers hold the cache as of the
    warm-up frame: the query cost does not depend on parameter values."""
    import dataclasses
    import multiprocessing as mp

    ref = _import_reference()
    if ref is None:
        return None
    from viscache import rng as RR
    from viscache.cache import MODE_LIGHTS as REF_LIGHTS, VisibilityCache as RefCache
    from viscache.hashgrid import HashGridConfig as RefGrid, init_params
    from viscache.mlp import AdamState, MLPConfig, he_init
    from viscache.render import make_gbuffer
    from viscache.scene import scene_from_dict as ref_scene
    from viscache.scenes import boxes_scene as ref_boxes
    from viscache.training import TrainFrameConfig as RefTF, train_frame as ref_train

    procs = procs or os.cpu_count() or 1
    s = ref_scene(ref_boxes(K))
    cam = dataclasses.replace(s.camera, width=WIDTH, height=HEIGHT)
    g = RefGrid(levels=LEVELS, table_size=TABLE, features_per_level=FEATS, aabb_min=s.aabb_min, aabb_max=s.aabb_max)
    c = RefCache(REF_LIGHTS, K, g, seed=0)
    # BASELINE's 3x64 MLP (the reference hardcodes (32, 32), cache.py:37-38): same
    # single init stream, table then He weights (cache.py:41-43)
    init = RR.stream(0, RR.INIT_PARAMS)
    c.grid_params = init_params(g, init)
    c.net_cfg = MLPConfig(input_dim=g.output_dim, output_dim=K, hidden_dims=HIDDEN)
    c.net_params = he_init(c.net_cfg, init)
    c.adam = AdamState.for_params(c._param_dict())
    tcfg = RefTF()
    t_setup = time.perf_counter()
    gb = make_gbuffer(s, cam)
    sel = np.arange(0, gb.n_pixels, every)
    pos, nrm, alb = (gb.flat(n)[sel] for n in ("position", "normal", "albedo"))
    for f in range(warmup):
        ref_train(s, cam, c, tcfg, frame=f)          # also JIT-compiles the numba kernels
    _REF_STATE.update(scene=s, cache=c, pos=pos, nrm=nrm, alb=alb)
    shards = [(int(a[0]), int(a[-1]) + 1) for a in np.array_split(np.arange(sel.size), procs) if a.size]
    t_train, t_query = [], []
    with mp.get_context("fork").Pool(len(shards)) as pool:
        pool.map(_ref_nls_shard, [(lo, hi, 0) for lo, hi in shards])   # per-camera tables + JIT, untimed
        setup_s = time.perf_counter() - t_setup
        for f in range(steps):
            t0 = time.perf_counter()
            ref_train(s, cam, c, tcfg, frame=warmup + f)
            t1 = time.perf_counter()
            pool.map(_ref_nls_shard, [(lo, hi, warmup + f) for lo, hi in shards])
            t2 = time.perf_counter()
            t_train.append(t1 - t0)
            t_query.append(t2 - t1)
    tr, q = statistics.median(t_train), statistics.median(t_query)
    p_total = WIDTH * HEIGHT
    frame_s = tr + q * (p_total / sel.size)
    return {"value": p_total / frame_s, "unit": UNIT, "cores": len(shards), "kind": "reference",
            "sample": (f"unmodified reference (baseline/_ref viscache 0.1.0, numpy+numba) on the host, median of "
                       f"{steps} steps: train_frame (8192 samples, 1 process) {tr:.2f} s + nls_sample_batch on "
                       f"every {every}th pixel ({sel.size} of {p_total}) over {len(shards)} processes "
                       f"{q:.2f} s, query extrapolated x{p_total / sel.size:.0f}; frame {frame_s:.2f} s "
                       f"(setup {setup_s:.0f} s untimed)"),
            "train_samples_per_s": (N_WORLD + N_SCREEN) / frame_s, "frame_s": frame_s,
            "train_s": tr, "query_sample_s": q, "steps": steps}


def cpu_baseline(steps: int = 3, warmup: int = 1) -> dict:
    """The reference when baseline/_ref is installed, else the oracle port."""
    cb = reference_cpu(steps=steps, warmup=warmup)
    return cb if cb is not None else cpu_reference()


REF_MAX_STEPS = 50


def reference_arm(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    # one reference step is ~0.7 s of host work: at most 50 steps keep the run
    # within a minute (the default --steps 1000 of the GPU arm would take ~12 min)
    cb = cpu_baseline(steps=min(args.steps, REF_MAX_STEPS), warmup=args.warmup)
    frame_s = cb["frame_s"]
    value = WIDTH * HEIGHT / frame_s
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": int(os.environ.get("WORLD_SIZE", "1")),
            "steps": cb.get("steps", args.steps), "warmup": args.warmup, "ms_per_step": frame_s * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f32 MLP / f64 index+WRS (numpy)",
            "data": "synthetic (boxes_scene(32) fixture, random-init weights, seed 0)",
            "config": {"workload": f"C2: {WIDTH}x{HEIGHT} boxes32 (K=32), L=16 T=2^19 F=2, MLP 3x64, "
                                   f"1 online frame = train batch {N_WORLD + N_SCREEN} (rows sharded over 1 ranks) "
                                   "+ NLS over all pixels",
                       "train_samples_per_s": (N_WORLD + N_SCREEN) / frame_s},
            "impl": "reference", "steps_requested": args.steps,
            "cpu_baseline": {k: cb[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main() -> None:
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)   # ~0.7 s timed: several in-region clock samples
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-sample", type=int, default=24576)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--workload", choices=["c2", "ndi4k", "render", "c4", "sweep", "clusters"], default="c2",
                    help="c2: the headline online frame (default); ndi4k: C3 Neural DI at 4K; "
                         "render: the c2 frame plus shading pass 5 (one shadow ray per pixel); "
                         "c4: the online frame on rooms128 with K=128 and a 3x128 MLP; "
                         "sweep: C5 query throughput over N = 2^16..2^26 and K = 8/32/128; "
                         "clusters: clustered NVC at 1080p with 1024 lights in 32 clusters")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        reference_arm(args)
    elif args.workload == "ndi4k":
        ndi4k_arm(args)
    elif args.workload == "sweep":
        sweep_arm(args)
    elif args.workload == "clusters":
        clusters_arm(args)
    else:
        gpu_arm(args)


if __name__ == "__main__":
    main()
