"""Profiling aid: achievable random-gather L2 bandwidth over the encoder's table footprint
(micro.cu nvc_l2_gather_probe), the denominator of the encoder's L2 roofline."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_05930_b200 import _lib  # noqa: E402

lib = _lib.load_micro()
entries = 16 * (1 << 19) * 2          # x-pair slots of the C2 table (8 B each, 67 MB)
table = torch.randint(0, 1 << 30, (entries * 2,), dtype=torch.int32, device="cuda")
sink = torch.zeros(1, dtype=torch.int64, device="cuda")
for grid, iters in ((148 * 8, 64), (148 * 16, 64), (148 * 32, 32)):
    for _ in range(2):
        lib.nvc_l2_gather_probe(table.data_ptr(), entries, grid, iters, sink.data_ptr(), None)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    lib.nvc_l2_gather_probe(table.data_ptr(), entries, grid, iters, sink.data_ptr(), None)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e)
    loads = grid * 256 * iters * 16
    print(f"grid {grid:5d}: {loads / ms / 1e6:8.1f} G gathers/s  payload {loads * 8 / ms / 1e6:7.1f} GB/s"
          f"  sectors {loads * 32 / ms / 1e6:8.1f} GB/s")
