"""Roofline denominators measured on this GPU (libnvc_micro.so):

* Philox4x64-10 block rate -- the integer-issue ceiling of the NLS kernel
  (generic 64-bit-counter blocks and the 32-bit-counter form it uses), plus a
  bit-equality check of the two forms;
* L2 streaming-read bandwidth over L2-resident buffers (16-B loads, .cg) --
  the encoder's L2 ceiling;
* the random 8-B gather rate over the encoder's 67 MB table (round 1's probe).

    python tools/rooflines.py            # prints one JSON object
Used by bench.py (measure()) so every bench line carries the denominators of
its own run."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def _time(fn, reps=3):
    import torch
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        best = min(best, s.elapsed_time(e))
    return best


def measure(quick: bool = False) -> dict:
    import torch
    from paper_2506_05930_b200 import _lib
    lib = _lib.load_micro()
    sms = torch.cuda.get_device_properties(0).multi_processor_count
    sink = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = torch.cuda.current_stream().cuda_stream     # the events below record on this stream
    out = {"sms": sms}
    key = 0x1234567890ABCDEF
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    lib.nvc_philox_check(key, 1 << 20, 1, bad.data_ptr(), st)
    lib.nvc_philox_check(key, 1 << 20, (1 << 32) - (1 << 20), bad.data_ptr(), st)
    torch.cuda.synchronize()
    out["philox_c32_equal"] = int(bad.item()) == 0
    for c32 in (0, 1):
        best = 0.0
        for per_sm in (8, 16, 32):
            grid, iters = sms * per_sm, 64 if quick else 256
            ms = _time(lambda: lib.nvc_philox_rate(c32, grid, iters, key, sink.data_ptr(), st))
            best = max(best, grid * 256 * iters / (ms * 1e-3))
        out["philox_blocks_per_s" + ("_c32" if c32 else "")] = best
    for mb in ((32, 64) if quick else (16, 32, 64)):
        buf = torch.randint(0, 1 << 30, (mb * (1 << 20) // 4,), dtype=torch.int32, device="cuda")
        best = 0.0
        for per_sm in (4, 8):
            grid, passes = sms * per_sm, 32     # >= 1 GB per launch: launch overhead is noise
            ms = _time(lambda: lib.nvc_l2_stream(buf.data_ptr(), buf.numel() * 4, grid, passes, sink.data_ptr(), st))
            best = max(best, buf.numel() * 4 * passes / (ms * 1e-3))
        out[f"l2_stream_GBps_{mb}MB"] = best / 1e9
        del buf
    entries = 16 * (1 << 19) * 2
    table = torch.randint(0, 1 << 30, (entries * 2,), dtype=torch.int32, device="cuda")
    grid, iters = sms * 16, 32 if quick else 64
    ms = _time(lambda: lib.nvc_l2_gather_probe(table.data_ptr(), entries, grid, iters, sink.data_ptr(), st))
    out["l2_gather_G_per_s_67MB"] = grid * 256 * iters * 16 / (ms * 1e-3) / 1e9
    return out


if __name__ == "__main__":
    print(json.dumps(measure()))
