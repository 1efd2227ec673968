"""The drop-in plugin's host logic, on CPU (no GPU needed): dropin.install()
rebinds exactly the reference's hot-path names and uninstall() restores them;
the NRC radiance cache (out of scope) stays the reference's CPU cache; light
and cluster caches are this package's and refuse to run without CUDA (there is
no CPU fallback).  Uses the unmodified reference in baseline/_ref
(tools/install_reference.sh); skipped where it is not installed."""

import importlib
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")
if not os.path.isdir(os.path.join(REF, "viscache")):
    pytest.skip("baseline/_ref (tools/install_reference.sh) is absent", allow_module_level=True)
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/nvc_numba_cache")
sys.path.insert(0, REF)

from paper_2506_05930_b200 import dropin  # noqa: E402
from paper_2506_05930_b200 import cache as our_cache  # noqa: E402


@pytest.fixture
def installed():
    dropin.install()
    yield
    dropin.uninstall()


def test_install_rebinds_and_uninstall_restores():
    mods = {m: importlib.import_module(m) for m in dropin.PATCHES}
    before = {(m, n): getattr(mods[m], n) for m, names in dropin.PATCHES.items() for n in names}
    dropin.install()
    try:
        for (m, n), fn in before.items():
            assert getattr(mods[m], n) is dropin.PATCHES[m][n], (m, n)
            assert getattr(mods[m], n) is not fn
        assert dropin.installed()
        dropin.install()                       # idempotent: originals are kept, not the patches
        assert all(dropin._ORIG[k] is v for k, v in before.items())
    finally:
        dropin.uninstall()
    for (m, n), fn in before.items():
        assert getattr(mods[m], n) is fn
    assert not dropin.installed()


def test_radiance_cache_stays_the_reference(installed):
    VR = importlib.import_module("viscache.render")
    from viscache.scene import scene_from_dict
    from viscache.scenes import boxes_scene
    s = scene_from_dict(boxes_scene(8))
    c = VR.make_cache(s, "radiance", seed=3)
    assert type(c).__module__ == "viscache.cache"
    assert c.infer(np.zeros((2, 3))).shape == (2, 3)        # the reference's numpy cache, on CPU


def test_light_cache_needs_cuda(installed):
    import torch
    if torch.cuda.is_available():
        pytest.skip("this checks the no-GPU behaviour")
    VR = importlib.import_module("viscache.render")
    from viscache.scene import scene_from_dict
    from viscache.scenes import boxes_scene
    s = scene_from_dict(boxes_scene(8))
    with pytest.raises(RuntimeError, match="CUDA"):
        VR.make_cache(s, "lights", seed=3)
    assert importlib.import_module("viscache.cache").VisibilityCache is our_cache.VisibilityCache
