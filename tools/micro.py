"""Profiling aid: tcgen05 MMA / TMEM-load latency microbenchmarks (micro.cu nvc_micro)."""
import ctypes, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2506_05930_b200 import _lib
lib = _lib.load_micro()
out = torch.zeros(1024, dtype=torch.int64, device="cuda")
def run(mode, iters, n, blocks):
    lib.nvc_micro(mode, iters, n, blocks, out.data_ptr(), None); torch.cuda.synchronize()
    lib.nvc_micro(mode, iters, n, blocks, out.data_ptr(), None); torch.cuda.synchronize()
    c = out[:blocks].float().mean().item()
    return c / iters
which = sys.argv[1] if len(sys.argv) > 1 else "all"
for n in ((32, 64, 128, 256) if which in ("all", "single") else ()):
    print(f"mode0 back-to-back MMA 128x{n}x16: {run(0, 4000, n, 1):.1f} cyc/MMA (1 CTA), {run(0, 4000, n, 148):.1f} (148 CTAs)")
if which in ("all", "single"):
  print(f"mode1 4xMMA(N=64)+commit+wait round trip: {run(1, 500, 64, 1):.0f} cyc (1 CTA)  {run(1, 500, 64, 296):.0f} (2/SM)")
  print(f"mode2 tcgen05.ld x16 + wait: {run(2, 2000, 64, 1):.1f} cyc")
_c = ctypes
lib.nvc_micro_multi.argtypes = [_c.c_int, _c.c_int, _c.c_int, _c.c_int, _c.c_void_p, _c.c_void_p]
lib.nvc_micro_pair.argtypes = [_c.c_int, _c.c_int, _c.c_int, _c.c_void_p, _c.c_void_p]
def run_multi(issuers, iters, n, blocks):
    for _ in range(2):
        lib.nvc_micro_multi(issuers, iters, n, blocks, out.data_ptr(), None); torch.cuda.synchronize()
    return out[:blocks].float().mean().item() / iters
def run_pair(iters, n, pairs):
    for _ in range(2):
        lib.nvc_micro_pair(iters, n, pairs, out.data_ptr(), None); torch.cuda.synchronize()
    return out[:2 * pairs:2].float().mean().item() / iters
for n in ((32, 64, 128) if which in ("all", "multi") else ()):
    print(f"multi-issuer 128x{n}x16, per issuer: " +
          ", ".join(f"{k} warps {run_multi(k, 2000, n, 1):.1f} cyc/MMA" for k in (1, 2, 4)))
for n in ((32, 64, 128, 256) if which in ("all", "pair") else ()):
    print(f"cta_group::2 256x{n}x16 back-to-back: {run_pair(4000, n, 1):.1f} cyc/MMA (1 pair), {run_pair(4000, n, 74):.1f} (74 pairs)")
