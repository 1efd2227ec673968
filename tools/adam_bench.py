"""Profiling aid: standalone time of the C2 Adam step (dense grid + MLP) for a given libnvc build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2506_05930_b200 import _lib  # noqa: E402

if len(sys.argv) > 1:
    _lib.load(sys.argv[1])
    _lib._lib = _lib.load(sys.argv[1])
from paper_2506_05930_b200 import MODE_LIGHTS, HashGridConfig, VisibilityCache  # noqa: E402

c = VisibilityCache(MODE_LIGHTS, 32, HashGridConfig(levels=16, table_size=1 << 19, features_per_level=2,
                                                    aabb_min=[-3, 0, -2.2], aabb_max=[3, 1.5, 3]),
                    hidden_dims=(64, 64, 64))
for _ in range(5):
    c.apply_adam()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(50):
    c.apply_adam()
e.record()
torch.cuda.synchronize()
print(f"{os.path.basename(sys.argv[1]) if len(sys.argv) > 1 else 'libnvc.so'} grid={os.environ.get('NVC_ADAM_GRID', 5)}: "
      f"{s.elapsed_time(e) / 50 * 1000:.1f} us per Adam step")
