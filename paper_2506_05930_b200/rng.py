"""Counter-based random streams, shared bit-for-bit with the reference.

The reference keys numpy's Philox4x64-10 with a splitmix64/FNV-1a fold of
(seed, frame, purpose, ...) parts (rng.py:30-56).  The CUDA kernels draw the
same stream by random access (draw n = lane n%4 of block n//4+1), so a
numpy ``Generator`` built by :func:`stream` and the GPU agree on every
uniform.  Sampling entry points accept either such a Generator (its position
is read, then advanced past the draws the GPU consumed) or a :class:`Stream`.
"""

from __future__ import annotations

import numpy as np

_M64 = (1 << 64) - 1

PRIMARY = "primary"
WORLD_SAMPLES = "world-samples"
SCREEN_SAMPLES = "screen-samples"
TARGETS = "targets"
LIGHT_SELECT = "light-select"
LIGHT_POINT = "light-point"
INIT_PARAMS = "init-params"
CLUSTERING = "clustering"


def _mix64(x: int) -> int:
    x = (x + 0x9E3779B97F4A7C15) & _M64
    for shift, mul in ((30, 0xBF58476D1CE4E5B9), (27, 0x94D049BB133111EB)):
        x = ((x ^ (x >> shift)) * mul) & _M64
    return x ^ (x >> 31)


def _fnv(text: str) -> int:
    h = 0xCBF29CE484222325
    for byte in text.encode("utf-8"):
        h = ((h ^ byte) * 0x100000001B3) & _M64
    return h


def stream_key(*parts) -> int:
    """64-bit key of a part tuple (strings hashed, ints masked to 64 bits)."""
    h = 0x8000000000000001
    for part in parts:
        h = _mix64(h ^ (_fnv(part) if isinstance(part, str) else part & _M64))
    return h


def stream(*parts) -> np.random.Generator:
    """numpy Generator for the key parts -- identical to the reference's."""
    return np.random.Generator(np.random.Philox(key=stream_key(*parts)))


class Stream:
    """Position in a keyed stream without host-side draws (device use)."""

    __slots__ = ("key", "offset")

    def __init__(self, *parts, key: int | None = None, offset: int = 0):
        self.key = stream_key(*parts) if key is None else int(key)
        self.offset = int(offset)

    def generator(self) -> np.random.Generator:
        g = np.random.Generator(np.random.Philox(key=self.key))
        set_position(g, self.offset)
        return g


def _philox_key(g: np.random.Generator) -> int:
    st = g.bit_generator.state
    if st.get("bit_generator") != "Philox":
        raise TypeError("light selection needs a Philox stream (rng.stream(...))")
    k = st["state"]["key"]
    if int(k[1]) != 0:
        raise TypeError("only 64-bit Philox keys are supported")
    return int(k[0])


def position(g) -> tuple[int, int]:
    """(key, number of draws already consumed) of a Generator or Stream."""
    if isinstance(g, Stream):
        return g.key, g.offset
    st = g.bit_generator.state
    key = _philox_key(g)
    c = st["state"]["counter"]
    ctr = int(c[0]) | (int(c[1]) << 64) | (int(c[2]) << 128) | (int(c[3]) << 192)
    if ctr == 0:
        return key, 0
    return key, (ctr - 1) * 4 + int(st["buffer_pos"])


def set_position(g: np.random.Generator, n: int) -> None:
    """Move a Philox Generator so its next draw is draw number n."""
    key = _philox_key(g)
    bg = np.random.Philox(key=key)
    if n > 0:
        blk, lane = divmod(n, 4)
        st = bg.state
        if lane == 0:
            st["state"]["counter"] = np.array([blk & _M64, blk >> 64, 0, 0], dtype=np.uint64)
            st["buffer_pos"] = 4
            bg.state = st
        else:
            st["state"]["counter"] = np.array([blk & _M64, blk >> 64, 0, 0], dtype=np.uint64)
            st["buffer_pos"] = 4
            bg.state = st
            bg.random_raw(lane)   # materialises block blk+1 and consumes `lane` words
    g.bit_generator.state = bg.state


def set_kept32(g: np.random.Generator, half) -> None:
    """Set the bit generator's kept 32-bit half (None: none) -- what numpy's
    32-bit draws (Generator.integers) leave behind for the next one."""
    st = g.bit_generator.state
    st["has_uint32"] = 0 if half is None else 1
    st["uinteger"] = 0 if half is None else int(half)
    g.bit_generator.state = st


def advance(g, n: int) -> None:
    """Account for n draws made on the device."""
    if isinstance(g, Stream):
        g.offset += int(n)
        return
    st = g.bit_generator.state
    kept = st["uinteger"] if st.get("has_uint32") else None   # 64-bit draws leave the kept half alone
    _, pos = position(g)
    set_position(g, pos + int(n))
    if kept is not None:
        set_kept32(g, kept)
