"""CPU tests of the host layer: scene fixtures, BVH, RNG plumbing, configs,
and the C ABI surface (library loads and exports every declared symbol)."""

import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

from paper_2506_05930_b200 import _lib
from paper_2506_05930_b200 import rng as R
from paper_2506_05930_b200.hashgrid import HashGridConfig
from paper_2506_05930_b200.mlp import TrainStepConfig, lr_at
from paper_2506_05930_b200.scene import Camera, build_bvh, camera_struct, scene_from_dict, shadow_epsilon
from paper_2506_05930_b200.scenes import boxes_point_scene, boxes_scene, rooms_scene

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "nvc.h")

SCENES = {"boxes8": lambda: boxes_scene(8), "boxes32": lambda: boxes_scene(32),
          "rooms128": lambda: rooms_scene(128), "pbox8": lambda: boxes_point_scene(8)}


@pytest.mark.parametrize("name", sorted(SCENES))
def test_scene_fixtures_match_reference(g_scenes, name):
    s = scene_from_dict(SCENES[name]())
    for k in ("v0", "v1", "v2"):
        np.testing.assert_array_equal(getattr(s, "triangles_" + k), g_scenes[f"{name}_{k}"])
    for k in ("tri_material", "tri_light", "lt_kind", "lt_verts", "lt_normal", "lt_area", "lt_radiance",
              "mat_albedo", "aabb_min", "aabb_max"):
        np.testing.assert_array_equal(getattr(s, k), g_scenes[f"{name}_{k}"])
    for k in ("node_min", "node_max", "node_left", "node_right", "node_start", "node_count", "perm"):
        np.testing.assert_array_equal(getattr(s.bvh, k), g_scenes[f"{name}_bvh_{k}"])


def test_empty_bvh():
    b = build_bvh(np.zeros((0, 3)), np.zeros((0, 3)), np.zeros((0, 3)))
    assert b.node_count[0] == 0 and shadow_epsilon(b) == pytest.approx(1e-4)


def test_scene_validation():
    from paper_2506_05930_b200.scene import SceneError
    d = boxes_scene(8)
    d["lights"] = []
    with pytest.raises(SceneError):
        scene_from_dict(d)
    with pytest.raises(ValueError):
        boxes_scene(7)
    with pytest.raises(ValueError):
        rooms_scene(33)


def test_stream_keys_match_reference(g_rng):
    parts = [(0,), (7,), (0, "init-params"), (0, 3, "light-select"), (5, 2, 1, "targets"), ("primary",),
             (123456789012345, -3, "x"), (2**64 - 1, 2**63)]
    assert [R.stream_key(*p) for p in parts] == [int(k) for k in g_rng["rng_keys"]]
    np.testing.assert_array_equal(R.stream(0, 3, "light-select").random(41), g_rng["rng_first"][3])


@pytest.mark.parametrize("n", [0, 1, 3, 4, 5, 17, 1001])
def test_generator_position_roundtrip(n):
    g = R.stream(1, 2, "light-select")
    g.random(n)
    key, pos = R.position(g)
    assert key == R.stream_key(1, 2, "light-select") and pos == n
    want = g.random(7)
    h = R.stream(1, 2, "light-select")
    R.set_position(h, n)
    np.testing.assert_array_equal(h.random(7), want)


def test_advance_matches_consumption():
    a, b = R.stream(4, "x"), R.stream(4, "x")
    a.random(10)
    R.advance(a, 23)
    b.random(33)
    np.testing.assert_array_equal(a.random(5), b.random(5))
    s = R.Stream(4, "x")
    R.advance(s, 33)
    np.testing.assert_array_equal(s.generator().random(5), R.stream(4, "x").random(38)[33:])


def test_grid_config_matches_reference(g_hash):
    for tag, levels, tsize in (("hc1", 8, 1 << 14), ("hc2", 16, 1 << 19)):
        c = HashGridConfig(levels=levels, table_size=tsize, features_per_level=2)
        assert [c.resolution(i) for i in range(levels)] == list(g_hash[tag + "_res"])
        assert [c.dense(i) for i in range(levels)] == list(g_hash[tag + "_dense"])
    with pytest.raises(ValueError):
        HashGridConfig(table_size=1000)
    with pytest.raises(ValueError):
        HashGridConfig(per_level_scale=1.0)


def test_lr_schedule():
    cfg = TrainStepConfig()
    assert lr_at(0, cfg) == 0.05 and lr_at(200, cfg) == pytest.approx(0.001)
    assert lr_at(100, cfg) == pytest.approx(0.0255)
    with pytest.raises(ValueError):
        lr_at(-1, cfg)


def test_camera_basis_struct():
    c = Camera([0, 1.25, 2.55], [0, 0, -0.9], [0, 1, 0], 48.0, 1920, 1080)
    s = camera_struct(c)
    fwd, right, up = c.basis()
    assert list(s.fwd) == list(fwd) and list(s.up) == list(up) and s.aspect == 1920 / 1080


def _declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(nvc_\w+)\s*\(", text, re.M)))


def test_header_and_binding_agree():
    assert set(_declared_symbols()) == set(_lib.EXPORTS)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in _declared_symbols():
        assert hasattr(lib, name), name
    assert lib.nvc_abi_version() == _lib.ABI_VERSION


def test_struct_layouts_match_c(tmp_path):
    src = tmp_path / "sz.c"
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "nvc.h"\nint main(void){'
                   'printf("%zu %zu %zu %zu %zu %zu %zu\\n", sizeof(nvc_model), sizeof(nvc_scene),'
                   ' sizeof(nvc_camera), offsetof(nvc_model, params), offsetof(nvc_scene, shadow_eps),'
                   ' offsetof(nvc_camera, width), offsetof(nvc_scene, anyhit_bf)); return 0; }\n')
    exe = tmp_path / "sz"
    subprocess.check_call(["gcc", "-I", os.path.dirname(HEADER), str(src), "-o", str(exe)])
    got = list(map(int, subprocess.check_output([str(exe)]).split()))
    want = [ctypes.sizeof(_lib.NvcModel), ctypes.sizeof(_lib.NvcScene), ctypes.sizeof(_lib.NvcCamera),
            _lib.NvcModel.params.offset, _lib.NvcScene.shadow_eps.offset, _lib.NvcCamera.width.offset,
            _lib.NvcScene.anyhit_bf.offset]
    assert got == want


@pytest.mark.parametrize("name", sorted(SCENES))
def test_shadow_accel_tables(name):
    """Per-triangle planes contain their triangle's vertices (to f32 rounding), every
    triangle's leaf holds it, and parent links walk from every leaf to the root."""
    from paper_2506_05930_b200.scene import shadow_accel
    b = scene_from_dict(SCENES[name]()).bvh
    plane, box, leaf, parent, r = shadow_accel(b)
    assert plane.dtype == np.float32 and plane.shape == (b.v0.shape[0], 4)
    live = np.abs(plane[:, :3]).sum(axis=1) > 0
    assert live.mean() > 0.9
    for v in (b.v0, b.v1, b.v2):
        resid = (plane[live, :3].astype(np.float64) * v[live]).sum(axis=1) - plane[live, 3]
        assert np.abs(resid).max() < 1e-5 * (1.0 + r)
    np.testing.assert_allclose(np.linalg.norm(plane[live, :3], axis=1), 1.0, rtol=1e-6)
    for v in (b.v0, b.v1, b.v2):
        assert (box[:, 0:3] <= v.astype(np.float32)).all() and (box[:, 4:7] >= v.astype(np.float32)).all()
    assert set(np.unique(box[:, 3])) <= {0.0, 1.0} and (box[:, 3] == 0).mean() > 0.9
    for k in range(b.v0.shape[0]):
        n = leaf[k]
        assert b.node_count[n] > 0 and b.node_start[n] <= k < b.node_start[n] + b.node_count[n]
        depth = 0
        while parent[n] >= 0:
            assert n in (b.node_left[parent[n]], b.node_right[parent[n]])
            n, depth = parent[n], depth + 1
        assert n == 0 and depth < 64
    assert r == max(np.abs(b.v0).max(), np.abs(b.v1).max(), np.abs(b.v2).max())


@pytest.mark.parametrize("tag,fn,k", [("r128k16", lambda: rooms_scene(128), 16), ("r1024k32", lambda: rooms_scene(1024), 32),
                                      ("b32k8", lambda: boxes_scene(32), 8), ("b8k8", lambda: boxes_scene(8), 8)])
def test_kmeans_matches_reference(g_clusters, tag, fn, k):
    """Light clustering (sampling.py:252-295): members, centroids and inertia history
    equal the reference's for the same "clustering" stream."""
    from paper_2506_05930_b200.clusters import kmeans_cluster
    cs = kmeans_cluster(scene_from_dict(fn()).lights, k, R.stream(0, R.CLUSTERING))
    np.testing.assert_array_equal(cs.centroids, g_clusters[f"km_{tag}_centroids"])
    np.testing.assert_array_equal([m.size for m in cs.members], g_clusters[f"km_{tag}_sizes"])
    np.testing.assert_array_equal(np.concatenate(cs.members), g_clusters[f"km_{tag}_members"])
    np.testing.assert_array_equal(cs.inertia_history, g_clusters[f"km_{tag}_history"])
    off, flat = cs.packed()
    assert off[-1] == flat.size == sum(m.size for m in cs.members)
    assert (cs.assignment[flat[off[3]:off[4]]] == 3).all()
    with pytest.raises(ValueError):
        kmeans_cluster(scene_from_dict(fn()).lights, 0, R.stream(0, R.CLUSTERING))


def test_no_device_means_loud_failure():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2506_05930_b200 import VisibilityCache
    with pytest.raises(RuntimeError, match="CUDA device"):
        VisibilityCache("lights", 8, HashGridConfig(levels=2, table_size=64))


def test_functional_api_surface():
    """The reference's module-level functions exist with its names; the host-only
    pieces (spatial_hash, init_params) agree with the reference formulas and the
    device ones fail loudly without a GPU."""
    import torch
    from paper_2506_05930_b200 import hashgrid as H
    from paper_2506_05930_b200 import mlp as M
    from paper_2506_05930_b200 import training as T
    for mod, names in ((H, ("init_params", "spatial_hash", "encode_batch", "encode", "grad_from_ctx", "encode_backward")),
                       (M, ("forward", "l2_loss", "backward_l2", "AdamState", "adam_step")),
                       (T, ("gen_screen_hits", "gen_screen_samples", "gen_world_samples"))):
        for n in names:
            assert callable(getattr(mod, n)), n
    c = np.array([[0, 0, 0], [1, 2, 3], [2**20, 7, 2**19]])
    np.testing.assert_array_equal(H.spatial_hash(c, 1 << 19),
                                  (c[:, 0] + c[:, 1] * 2654435761 + c[:, 2] * 805459861) & ((1 << 19) - 1))
    cfg = HashGridConfig(levels=2, table_size=64)
    t = H.init_params(cfg, R.stream(0, "init-params"))
    assert t.shape == (2, 64, 4) and t.dtype == np.float32 and np.abs(t).max() <= 1e-4
    np.testing.assert_array_equal(t, R.stream(0, "init-params").uniform(-1e-4, 1e-4, (2, 64, 4)).astype(np.float32))
    st = M.AdamState.for_params({"w": np.ones(3, np.float32)})
    assert st.t == 0 and st.beta1 == 0.9 and st.beta2 == 0.999 and st.eps == 1e-8
    if not torch.cuda.is_available():
        with pytest.raises(RuntimeError, match="CUDA device"):
            H.encode_batch(np.zeros((1, 3)), cfg, t)
        with pytest.raises(RuntimeError, match="CUDA device"):
            M.forward(M.he_init(M.MLPConfig(4, 2), R.stream(0, "x")), M.MLPConfig(4, 2), np.zeros((1, 4), np.float32))
