"""G-buffer (render pass 1) and the per-camera pixel context, on the GPU.

Mirrors ``viscache.render.make_gbuffer`` / ``gbuffer_and_ctx``
(render.py:49-142): primary rays jittered by the ("primary",) stream with
draws (2p, 2p+1), FP64 closest hit against the reference-ordered BVH, facing
normals and material albedo -- bit-identical to the reference.  The
light-major factor/luminance tables of the returned PixelCtx are memoized
per camera exactly like the reference memoizes its P x K matrices.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from . import rng as rngmod
from .sampling import PixelCtx
from .scene import camera_struct, device_scene


@dataclass
class GBuffer:
    width: int
    height: int
    hit: object
    position: object
    normal: object
    albedo: object
    light_id: object

    @property
    def shape(self):
        return (self.height, self.width)

    @property
    def n_pixels(self) -> int:
        return self.width * self.height

    def flat(self, name: str):
        a = getattr(self, name)
        return a.reshape(self.n_pixels, *a.shape[2:])


def gbuffer_device(scene, camera=None, p_first: int = 0, p_count: int | None = None, device=None):
    """(pos, nrm, alb, hit, light_id) CUDA tensors for pixels [p_first, p_first+p_count)."""
    import torch
    camera = camera or scene.camera
    ds = device_scene(scene, device)
    p = camera.width * camera.height - p_first if p_count is None else p_count
    dev = ds.device
    pos = torch.empty((p, 3), dtype=torch.float64, device=dev)
    nrm = torch.empty((p, 3), dtype=torch.float64, device=dev)
    alb = torch.empty((p, 3), dtype=torch.float64, device=dev)
    hit = torch.empty(p, dtype=torch.uint8, device=dev)
    lid = torch.empty(p, dtype=torch.int32, device=dev)
    _lib.call("nvc_gbuffer", ds.struct, camera_struct(camera), rngmod.stream_key(rngmod.PRIMARY), p_first, p,
              pos.data_ptr(), nrm.data_ptr(), alb.data_ptr(), hit.data_ptr(), lid.data_ptr(), _lib.stream_ptr())
    return pos, nrm, alb, hit, lid


def make_gbuffer(scene, camera=None) -> GBuffer:
    camera = camera or scene.camera
    w, h = camera.width, camera.height
    pos, nrm, alb, hit, lid = (t.cpu().numpy() for t in gbuffer_device(scene, camera))
    return GBuffer(w, h, hit.astype(bool).reshape(h, w), pos.reshape(h, w, 3), nrm.reshape(h, w, 3),
                   alb.reshape(h, w, 3), lid.reshape(h, w))


def gbuffer_and_ctx(scene, camera=None, table_dtype=np.float32):
    """Device PixelCtx over all pixels, memoized on the scene per camera."""
    camera = camera or scene.camera
    key = ("gbuf", camera.width, camera.height, tuple(camera.position), tuple(camera.look_at),
           camera.fov_deg, np.dtype(table_dtype).str)
    memo = scene.__dict__.setdefault("_nvc_memo", {})
    if key not in memo:
        pos, nrm, alb, hit, lid = gbuffer_device(scene, camera)
        ctx = PixelCtx(scene, pos, nrm, alb, table_dtype=table_dtype)
        ctx.hit, ctx.light_id = hit, lid
        memo[key] = ctx
    return memo[key]
