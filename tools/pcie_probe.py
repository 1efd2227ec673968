"""Profiling aid: pinned host<->device copy bandwidth (one direction, and both at once)."""
import time

import torch

n = 50_000_000 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, reps=20):
    for it in range(reps + 3):
        if it == 3:
            torch.cuda.synchronize()
            t = time.perf_counter()
        if h2d:
            with torch.cuda.stream(s1):
                d.copy_(h, non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    return n * 8 * reps / (time.perf_counter() - t) / 1e9


print(f"H2D alone: {run(True, False):.1f} GB/s")
print(f"D2H alone: {run(False, True):.1f} GB/s")
print(f"both at once: {run(True, True):.1f} GB/s each way")
