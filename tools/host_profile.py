"""Profiling aid: where the host spends its time enqueueing C2 frames (cProfile)."""
import cProfile
import os
import pstats
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402

sys.argv = ["bench.py", "--steps", "300", "--warmup", "3", "--no-cpu-baseline"]
pr = cProfile.Profile()
pr.enable()
bench.main()
pr.disable()
st = pstats.Stats(pr)
st.sort_stats("cumulative").print_stats("frame_into|train_frame_device|nls_sample_device|release|_launch|gen_batch_device|camera_struct|device_scene")
st.print_callers("from_callable|_lib.py:153")
