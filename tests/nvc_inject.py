"""pytest plugin: run the reference's OWN test suite against the CUDA cache.

    PYTHONPATH=tests:. python -m pytest -p nvc_inject baseline/_ref/viscache_tests/test_sampling.py

Before the reference's test modules are imported, ``dropin.install()`` rebinds
the reference's hot-path names (VisibilityCache, make_cache, train_frame,
nls_sample_batch, nls_weights_batch, neural_di_batch, clustered_sample_batch,
gbuffer_and_ctx, shade_batch) to this package's CUDA versions, so every test
that builds a cache, trains it or samples lights through those names runs on
the GPU.  baseline/_ref is the unmodified reference installed by
tools/install_reference.sh (it travels to the GPU box with the snapshot).
NVC_INJECT_PRECISION=fp32 makes the injected caches infer on the f32 SIMT
parity path instead of the fp16 tcgen05 default.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")


def pytest_configure(config):
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nvc_numba_cache")
    for p in (ROOT, REF):
        if p not in sys.path:
            sys.path.insert(0, p)
    import viscache  # noqa: F401  (the reference, from baseline/_ref)
    from paper_2506_05930_b200 import PRECISION_FP16, PRECISION_FP32, dropin
    prec = PRECISION_FP32 if os.environ.get("NVC_INJECT_PRECISION") == "fp32" else PRECISION_FP16
    dropin.install(precision=prec)
    config.addinivalue_line("markers", "nvc_injected: the reference suite runs on the CUDA cache")


def pytest_terminal_summary(terminalreporter):
    from paper_2506_05930_b200 import _lib, dropin
    terminalreporter.write_line(f"nvc_inject: reference names rebound to paper_2506_05930_b200: "
                                f"{len(dropin._ORIG)} (libnvc: {_lib.load()._name})")
