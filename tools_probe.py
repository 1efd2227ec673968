import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import torch
from paper_2506_05930_b200 import _lib, MODE_LIGHTS, HashGridConfig, VisibilityCache, PRECISION_FP16
from paper_2506_05930_b200.render import gbuffer_device
from paper_2506_05930_b200.scene import scene_from_dict
from paper_2506_05930_b200.scenes import boxes_scene
lib = _lib.load()
lib.nvc_encode_probe.argtypes = [ctypes.POINTER(_lib.NvcModel), ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p]
scene = scene_from_dict(boxes_scene(32))
cam = scene.camera.resized(1920, 1080)
pos, nrm, alb, _, _ = gbuffer_device(scene, cam)
grid = HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2, aabb_min=scene.aabb_min, aabb_max=scene.aabb_max)
cache = VisibilityCache(MODE_LIGHTS, 32, grid, hidden_dims=(64, 64, 64))
P = pos.shape[0]
feats = torch.empty((P, 32), dtype=torch.float16, device="cuda")
vis = torch.empty((P, 32), dtype=torch.float32, device="cuda")
def t(fn, n=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n * 1000
print("encode probe (thread per pixel-level): %.1f us" % t(lambda: lib.nvc_encode_probe(cache.model, pos.data_ptr(), P, feats.data_ptr(), None)))
print("infer fp16 fused (flat, vis mode): %.1f us" % t(lambda: cache.infer_device(pos, PRECISION_FP16, out=vis)))
for d in ("1", "12", "13"):
    os.environ["NVC_QUERY_DEBUG"] = d
    print("infer fp16 fused dbg=%s: %.1f us" % (d, t(lambda: cache.infer_device(pos, PRECISION_FP16, out=vis))))
