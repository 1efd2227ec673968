"""paper_2506_05930_b200 -- B200-native neural visibility cache (arXiv 2506.05930).

A drop-in for the hot path of the reference ``viscache`` package: the cache
object (``VisibilityCache``/``make_cache`` with ``infer``/``train_step``),
the training-frame driver, WRS light sampling / Neural DI and the
one-shadow-ray shading pass.  All compute
runs in ``libnvc.so`` (hand-written sm_100a CUDA: FP64 geometry, hash-grid
encoder, tcgen05/TMEM fused MLP, WRS with numpy-compatible Philox); this
package is the host layer that keeps the reference's API.
"""

from . import rng
from .cache import (MODE_CLUSTERS, MODE_LIGHTS, MODE_RADIANCE, PRECISION_FP16, PRECISION_FP32,
                    GradExchange, VisibilityCache, make_cache)
from .hashgrid import HashGridConfig, clustered_config
from .mlp import MLPConfig, MLPParams, TrainStepConfig, lr_at
from . import render
from .render import GBuffer, gbuffer_and_ctx, make_gbuffer, shade_batch, shade_pixel
from .clusters import ClusterSet, kmeans_cluster
from .sampling import (CLAMP_FLOOR, PixelCtx, Reservoir, ShadingPoint, clamp_visibility, clustered_sample,
                       clustered_sample_batch,
                       neural_di_batch, neural_di_shade, nls_sample, nls_sample_batch,
                       nls_weights_batch, wrs_select, wrs_select_batch)
from .scene import Camera, Light, Material, Scene, SceneError, load_scene, scene_from_dict
from .scenes import boxes_point_scene, boxes_scene, rooms_scene
from .training import (TrainFrameConfig, compute_visibility_targets, gen_screen_hits, gen_screen_samples,
                       gen_world_samples, train_frame)
from . import restir
from .restir import (ReservoirGrid, cnvc_initial_batch, restir_spatial_batch, restir_temporal_batch,
                     ris_initial_batch)
from . import dropin

__version__ = "0.1.0"

__all__ = [
    "rng", "VisibilityCache", "make_cache", "MODE_LIGHTS", "MODE_CLUSTERS", "MODE_RADIANCE",
    "PRECISION_FP16", "PRECISION_FP32", "HashGridConfig", "clustered_config", "MLPConfig",
    "MLPParams", "TrainStepConfig", "lr_at", "GBuffer", "gbuffer_and_ctx", "make_gbuffer", "render",
    "shade_batch", "shade_pixel",
    "CLAMP_FLOOR", "PixelCtx", "Reservoir", "ShadingPoint", "clamp_visibility", "neural_di_batch",
    "neural_di_shade", "nls_sample", "nls_sample_batch", "nls_weights_batch", "wrs_select",
    "wrs_select_batch", "Camera", "Light", "Material", "Scene", "SceneError", "load_scene",
    "scene_from_dict", "boxes_scene", "boxes_point_scene", "rooms_scene", "TrainFrameConfig",
    "compute_visibility_targets", "gen_screen_hits", "gen_screen_samples", "gen_world_samples", "train_frame",
    "ClusterSet", "kmeans_cluster", "clustered_sample", "clustered_sample_batch", "dropin",
    "restir", "ReservoirGrid", "ris_initial_batch", "restir_temporal_batch", "restir_spatial_batch",
    "cnvc_initial_batch",
]
