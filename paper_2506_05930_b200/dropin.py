"""Reference plugin: run the reference package's own frame loop on this cache.

The reference has no C ABI or registry for the visibility-cache path; its
"plugin interface" is a duck-typed cache object plus a handful of module-level
functions that its frame loop looks up at call time (
``render_frame``, render.py:283-375).  ``install()`` rebinds exactly those
names in the imported ``viscache`` modules to this package's CUDA versions:

====================================  ========================================
reference name (file:line)            replaced by
====================================  ========================================
cache.VisibilityCache (cache.py:25)   cache.VisibilityCache (device params)
cache/render.make_cache (:120-139)    make_cache below (radiance mode -> ref)
training/render.train_frame (:166)    train_frame below (other caches -> ref)
sampling/render.nls_sample_batch      sampling.nls_sample_batch
sampling.nls_weights_batch            sampling.nls_weights_batch
sampling/render.neural_di_batch       sampling.neural_di_batch
sampling/render.clustered_sample_batch sampling.clustered_sample_batch
render.gbuffer_and_ctx (:128-142)     render.gbuffer_and_ctx ((gb, ctx))
render.shade_batch (:220-246)         render.shade_batch (k_shade)
sampling/render.ris_initial_batch,    restir.* (nvc_ris_initial,
  cnvc_initial_batch,                   nvc_restir_temporal,
  restir_temporal/spatial_batch         nvc_restir_spatial)
====================================  ========================================

Everything else -- scenes, cameras, configs, ``ClusterSet`` / k-means, the
ReSTIR/RIS and NRC baselines, metrics, I/O -- stays the reference's.  Its
objects are accepted as they are: scenes, cameras and configs are read by
attribute (the same fields), a reference ``PixelCtx`` is wrapped on the device
once per camera (``sampling.as_pixel_ctx``), a reference ``ClusterSet`` is
read through ``members``.  A cache that is not this package's (a test double,
the NRC radiance cache) goes to the reference's own functions or, for the
sampling kernels, through ``cache.infer``.

    import viscache
    from paper_2506_05930_b200 import dropin
    dropin.install()          # reference render_frame now runs on the GPU
    ...
    dropin.uninstall()
"""

from __future__ import annotations

import importlib

import numpy as np

from . import cache as _cache
from . import render as _render
from . import restir as _restir
from . import sampling as _sampling
from . import training as _training

_ORIG: dict = {}
_DEFAULTS: dict = {}     # extra VisibilityCache kwargs for caches make_cache builds (e.g. precision)


def _ref(modname: str, name: str):
    return _ORIG.get((modname, name)) or getattr(importlib.import_module(modname), name)


def make_cache(scene, mode, seed=0, clusters=None, grid=None, train=None, dtype=np.float32, **kw):
    """reference make_cache (cache.py:120-139): the CUDA cache for light and
    cluster outputs; the NRC radiance baseline (out of scope) stays the
    reference's CPU cache."""
    if mode == _cache.MODE_RADIANCE:
        # the reference's own cache class (viscache.cache.VisibilityCache is rebound)
        from viscache.hashgrid import HashGridConfig as RefGrid
        grid = grid or RefGrid(aabb_min=scene.aabb_min, aabb_max=scene.aabb_max)
        return _ref("viscache.cache", "VisibilityCache")(mode, 3, grid, train=train, seed=seed, dtype=dtype)
    return _cache.make_cache(scene, mode, seed=seed, clusters=clusters, grid=grid, train=train, dtype=dtype,
                             **{**_DEFAULTS, **kw})


def train_frame(scene, camera, cache, cfg, frame=0, clusters=None):
    """reference train_frame (training.py:166-199) on the device for this
    package's cache; any other cache object trains through the reference."""
    if isinstance(cache, _cache.VisibilityCache):
        return _training.train_frame(scene, camera, cache, cfg, frame=frame, clusters=clusters)
    return _ref("viscache.training", "train_frame")(scene, camera, cache, cfg, frame=frame, clusters=clusters)


PATCHES = {
    "viscache.cache": {"VisibilityCache": _cache.VisibilityCache, "make_cache": make_cache},
    "viscache.training": {"train_frame": train_frame},
    "viscache.sampling": {"nls_sample_batch": _sampling.nls_sample_batch,
                          "nls_weights_batch": _sampling.nls_weights_batch,
                          "neural_di_batch": _sampling.neural_di_batch,
                          "clustered_sample_batch": _sampling.clustered_sample_batch,
                          "ris_initial_batch": _restir.ris_initial_batch,
                          "cnvc_initial_batch": _restir.cnvc_initial_batch,
                          "restir_temporal_batch": _restir.restir_temporal_batch,
                          "restir_spatial_batch": _restir.restir_spatial_batch},
    "viscache.render": {"make_cache": make_cache, "train_frame": train_frame,
                        "nls_sample_batch": _sampling.nls_sample_batch,
                        "neural_di_batch": _sampling.neural_di_batch,
                        "clustered_sample_batch": _sampling.clustered_sample_batch,
                        "gbuffer_and_ctx": _render.gbuffer_and_ctx,
                        "shade_batch": _render.shade_batch,
                        "ris_initial_batch": _restir.ris_initial_batch,
                        "cnvc_initial_batch": _restir.cnvc_initial_batch,
                        "restir_temporal_batch": _restir.restir_temporal_batch,
                        "restir_spatial_batch": _restir.restir_spatial_batch,
                        "ReservoirGrid": _restir.ReservoirGrid},
}


def install(patches: dict | None = None, **cache_kw) -> dict:
    """Rebind the reference names (idempotent); returns {(module, name): original}.
    ``cache_kw`` (e.g. ``precision=PRECISION_FP32``) go to every cache the
    injected make_cache builds."""
    _DEFAULTS.clear()
    _DEFAULTS.update(cache_kw)
    for modname, names in (patches or PATCHES).items():
        mod = importlib.import_module(modname)
        for name, fn in names.items():
            _ORIG.setdefault((modname, name), getattr(mod, name))
            setattr(mod, name, fn)
    return dict(_ORIG)


def uninstall() -> None:
    for (modname, name), fn in _ORIG.items():
        setattr(importlib.import_module(modname), name, fn)
    _ORIG.clear()
    _DEFAULTS.clear()


def installed() -> bool:
    return bool(_ORIG)


__all__ = ["install", "uninstall", "installed", "make_cache", "train_frame", "PATCHES"]
