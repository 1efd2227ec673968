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
    """The reference's G-buffer (render.py:79-100): (h, w[, 3]) host arrays."""

    width: int
    height: int
    hit: object
    position: object
    normal: object
    albedo: object
    depth: object
    light_id: object
    emissive: object

    @property
    def shape(self):
        return (self.height, self.width)

    @property
    def n_pixels(self) -> int:
        return self.width * self.height

    def flat(self, name: str):
        a = getattr(self, name)
        return a.reshape(self.n_pixels, *a.shape[2:])


def gbuffer_device(scene, camera=None, p_first: int = 0, p_count: int | None = None, device=None,
                   full: bool = False):
    """(pos, nrm, alb, hit, light_id) CUDA tensors for pixels [p_first, p_first+p_count);
    with ``full`` also (depth, emissive)."""
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
    depth = torch.empty(p, dtype=torch.float64, device=dev) if full else None
    emis = torch.empty((p, 3), dtype=torch.float64, device=dev) if full else None
    _lib.call("nvc_gbuffer", ds.struct, camera_struct(camera), rngmod.stream_key(rngmod.PRIMARY), p_first, p,
              pos.data_ptr(), nrm.data_ptr(), alb.data_ptr(), hit.data_ptr(), lid.data_ptr(), _lib.ptr(depth),
              _lib.ptr(emis), _lib.stream_ptr())
    return (pos, nrm, alb, hit, lid, depth, emis) if full else (pos, nrm, alb, hit, lid)


def _gbuffer_host(camera, pos, nrm, alb, hit, lid, depth, emis) -> GBuffer:
    w, h = camera.width, camera.height
    pos, nrm, alb, hit, lid, depth, emis = (t.cpu().numpy() for t in (pos, nrm, alb, hit, lid, depth, emis))
    return GBuffer(w, h, hit.astype(bool).reshape(h, w), pos.reshape(h, w, 3), nrm.reshape(h, w, 3),
                   alb.reshape(h, w, 3), depth.reshape(h, w), lid.astype(np.int64).reshape(h, w),
                   emis.reshape(h, w, 3))


def make_gbuffer(scene, camera=None) -> GBuffer:
    """Primary-ray G-buffer (render.py:103-117), bit-identical to the reference."""
    camera = camera or scene.camera
    return _gbuffer_host(camera, *gbuffer_device(scene, camera, full=True))


def gbuffer_and_ctx(scene, camera=None, table_dtype=np.float64):
    """(G-buffer, PixelCtx over all pixels), memoized on the scene per camera
    (render.py:128-142).  The G-buffer is host-side like the reference's; the
    PixelCtx keeps its positions / normals / albedos and its light-major
    factor and luminance tables on the device (``table_dtype`` float64 is the
    reference's precision; float32 halves the hot loop's table traffic)."""
    camera = camera or scene.camera
    key = ("gbuf", camera.width, camera.height, tuple(camera.position), tuple(camera.look_at),
           camera.fov_deg, np.dtype(table_dtype).str)
    memo = scene.__dict__.setdefault("_nvc_memo", {})
    if key not in memo:
        pos, nrm, alb, hit, lid, depth, emis = gbuffer_device(scene, camera, full=True)
        ctx = PixelCtx(scene, pos, nrm, alb, table_dtype=table_dtype)
        ctx.hit, ctx.light_id = hit, lid
        memo[key] = (_gbuffer_host(camera, pos, nrm, alb, hit, lid, depth, emis), ctx)
    return memo[key]


# ---------------------------------------------------------------------------
# Shading pass 5 (render.py:220-246): one shadow ray per pixel
# ---------------------------------------------------------------------------

def shade_device(scene, positions, normals, albedos, ids, points, big_w, out=None):
    """``shade_batch`` on CUDA tensors (pos/nrm/alb/points (n,3) f64, ids (n) i64,
    big_w (n) f64, all on the scene's device): rgb (n,3) f64, bit-identical to the
    reference.  Launches ``k_shade`` on the current stream, no host sync."""
    import torch
    ds = device_scene(scene, positions.device)
    n = positions.shape[0]
    if out is None:
        out = torch.empty((n, 3), dtype=torch.float64, device=positions.device)
    args = [t.contiguous() for t in (positions, normals, albedos, ids, points, big_w)]
    if args[3].dtype != torch.int64 or any(a.dtype != torch.float64 for i, a in enumerate(args) if i != 3):
        raise TypeError("shade_device: f64 positions/normals/albedos/points/big_w and int64 ids expected")
    _lib.call("nvc_shade", ds.struct, *(a.data_ptr() for a in args), n, out.data_ptr(), _lib.stream_ptr())
    return out


def shade_batch(scene, positions, normals, albedos, ids, points, big_w):
    """One-shadow-ray area-measure estimate per row:
    albedo/pi * L_e * G * V * area * W (point lights drop the area term).

    Same signature and result as the reference's ``shade_batch``; numpy in ->
    numpy out (via the device), CUDA tensors in -> CUDA tensor out."""
    torch = _lib.require_cuda()
    if isinstance(positions, torch.Tensor) and positions.is_cuda:
        return shade_device(scene, positions, normals, albedos, ids, points, big_w)
    dev = device_scene(scene).device
    f64 = lambda a: torch.from_numpy(np.ascontiguousarray(np.atleast_2d(a), np.float64)).to(dev)  # noqa: E731
    ids_t = torch.from_numpy(np.ascontiguousarray(np.atleast_1d(ids), np.int64)).to(dev)
    w_t = torch.from_numpy(np.ascontiguousarray(np.atleast_1d(big_w), np.float64)).to(dev)
    out = shade_device(scene, f64(positions), f64(normals), f64(albedos), ids_t, f64(points), w_t)
    return out.cpu().numpy()


def shade_pixel(sp, light_sample, scene) -> np.ndarray:
    """Scalar shading of one (light id, point, W) sample (render.py:249-256)."""
    lid, point, big_w = light_sample
    if big_w < 0:
        raise ValueError("contribution weight must be nonnegative")
    return shade_batch(scene, np.asarray(sp.position)[None], np.asarray(sp.normal)[None],
                       np.asarray(sp.albedo)[None], np.array([lid]), np.atleast_2d(point), np.array([big_w]))[0]
