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
for n in (32, 64, 128, 256):
    print(f"mode0 back-to-back MMA 128x{n}x16: {run(0, 4000, n, 1):.1f} cyc/MMA (1 CTA), {run(0, 4000, n, 148):.1f} (148 CTAs)")
print(f"mode1 4xMMA(N=64)+commit+wait round trip: {run(1, 500, 64, 1):.0f} cyc (1 CTA)  {run(1, 500, 64, 296):.0f} (2/SM)")
print(f"mode2 tcgen05.ld x16 + wait: {run(2, 2000, 64, 1):.1f} cyc")
