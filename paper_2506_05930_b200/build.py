"""Build libnvc.so (all CUDA for sm_100a) in-tree.

    python -m paper_2506_05930_b200.build        # or __graft_entry__.build()

geometry.cu is compiled with -fmad=false (bit-exact FP64 geometry, no FMA
contraction); the other TUs use explicit __*_rn intrinsics wherever the
reference's rounding must be reproduced, so they keep FMA elsewhere.
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libnvc.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "--expt-relaxed-constexpr",
                 "-I", os.path.join(HERE, "..", "include")]
UNITS = {"geometry.cu": ["-fmad=false"], "model.cu": [], "query.cu": [], "pipeline.cu": []}
MICRO_OUT = os.path.join(HERE, "libnvc_micro.so")     # microbenchmarks (tools/, bench rooflines)


def nvcc() -> str:
    cand = os.path.join(os.environ.get("CUDA_HOME", "/usr/local/cuda"), "bin", "nvcc")
    return cand if os.path.exists(cand) else "nvcc"


def build(verbose: bool = False, force: bool = False, defs: list[str] | None = None, out: str = OUT) -> str:
    """defs: extra -D flags (profiling builds, e.g. ["-DNVC_TRACE"] -> a separate .so)."""
    defs = defs or []
    objdir = os.path.join(HERE, "build" + ("_" + "_".join(d.lstrip("-D").lower() for d in defs) if defs else ""))
    os.makedirs(objdir, exist_ok=True)
    deps = [os.path.join(CSRC, f) for f in os.listdir(CSRC)] + [os.path.join(HERE, "..", "include", "nvc.h")]
    newest = max(os.path.getmtime(d) for d in deps)
    if not force and os.path.exists(out) and os.path.getmtime(out) >= newest:
        return out
    objs = []
    for unit, extra in UNITS.items():
        obj = os.path.join(objdir, unit.replace(".cu", ".o"))
        cmd = [nvcc(), *COMMON, *extra, *defs, "-c", os.path.join(CSRC, unit), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
            print(" ".join(cmd))
        subprocess.check_call(cmd)
        objs.append(obj)
    tmp = out + ".tmp"
    subprocess.check_call([nvcc(), *ARCH, "-shared", "-cudart", "static", "-o", tmp, *objs])
    os.replace(tmp, out)
    return out


def build_micro(force: bool = False, out: str = MICRO_OUT) -> str:
    """libnvc_micro.so: csrc/micro.cu alone (roofline-denominator microbenchmarks)."""
    src = os.path.join(CSRC, "micro.cu")
    deps = [src, os.path.join(CSRC, "common.cuh"), os.path.join(HERE, "..", "include", "nvc.h")]
    if not force and os.path.exists(out) and os.path.getmtime(out) >= max(os.path.getmtime(d) for d in deps):
        return out
    tmp = out + ".tmp"
    subprocess.check_call([nvcc(), *COMMON, "-DNVC_MICRO_STANDALONE", "-shared", "-cudart", "static", src, "-o", tmp])
    os.replace(tmp, out)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv, force=True))
    print(build_micro(force=True))
