import ctypes, os, sys, json
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
os.environ.setdefault("NVC_QUERY_DEBUG", "128")
from paper_2506_05930_b200 import _lib, MODE_LIGHTS, HashGridConfig, VisibilityCache
from paper_2506_05930_b200 import rng as R
from paper_2506_05930_b200.render import gbuffer_device
from paper_2506_05930_b200.sampling import PixelCtx, nls_sample_device
from paper_2506_05930_b200.scene import scene_from_dict
from paper_2506_05930_b200.scenes import boxes_scene
lib = _lib.load()
lib.nvc_debug_trace.restype = ctypes.c_int
lib.nvc_debug_trace.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32]
scene = scene_from_dict(boxes_scene(32))
cam = scene.camera.resized(1920, 1080)
pos, nrm, alb, _, _ = gbuffer_device(scene, cam)
ctx = PixelCtx(scene, pos, nrm, alb); ctx.lum_device(); ctx.mask_device("lum")
grid = HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2, aabb_min=scene.aabb_min, aabb_max=scene.aabb_max)
cache = VisibilityCache(MODE_LIGHTS, 32, grid, hidden_dims=(64, 64, 64))
for i in range(3):
    nls_sample_device(ctx, cache, R.stream_key(0, i, "light-select"))
torch.cuda.synchronize()
lib.nvc_debug_trace(None, 0, 1)
nls_sample_device(ctx, cache, R.stream_key(0, 9, "light-select"))
torch.cuda.synchronize()
buf = (ctypes.c_uint64 * 8192)()
n = lib.nvc_debug_trace(ctypes.addressof(buf), 8192, 0)
ev = sorted((int(b) >> 16, int(b) & 0xffff) for b in buf[:n])
t0 = ev[0][0]
names = {1: "tile start", 2: "encode done", 3: "after sync", 4: "mma issued", 5: "mma done", 6: "epi done", 7: "epi synced", 8: "final done", 9: "outputs done"}
out = [f"{(t - t0):9d} cyc  {names.get(c >> 8, c >> 8)} l={(c >> 4) & 15} s={c & 15}" for t, c in ev]
open("gpurun_out/trace.txt", "w").write("\n".join(out))
print(n, "events")
