"""ctypes binding of libnvc.so (include/nvc.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every compute entry point raises.  Device buffers are
torch tensors; only their raw pointers cross the C ABI.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libnvc.so")

MAX_LEVELS = 32
MAX_LAYERS = 8
ABI_VERSION = 11

c_i32, c_i64, c_u64, c_f64, c_f32, c_vp = (ctypes.c_int32, ctypes.c_int64, ctypes.c_uint64,
                                           ctypes.c_double, ctypes.c_float, ctypes.c_void_p)


class NvcModel(ctypes.Structure):
    _fields_ = [
        ("levels", c_i32), ("features", c_i32), ("table_size", c_i64),
        ("resolution", c_i32 * MAX_LEVELS), ("dense", c_i32 * MAX_LEVELS),
        ("aabb_min", c_f64 * 3), ("span", c_f64 * 3),
        ("n_layers", c_i32), ("dims", c_i32 * (MAX_LAYERS + 1)),
        ("alpha", c_f32), ("out_sigmoid", c_i32),
        ("params", c_vp), ("adam_m", c_vp), ("adam_v", c_vp), ("grad_fx", c_vp),
        ("touch_bits", c_vp), ("touch_off", c_vp), ("grad_c", c_vp), ("grad_c_entries", c_i64),
        ("table_h", c_vp), ("wpack", c_vp),
        ("param_count", c_i64), ("wpack_count", c_i64),
    ]


class NvcRGrid(ctypes.Structure):
    _fields_ = [("y", c_vp), ("point", c_vp), ("w_y", c_vp), ("w_sum", c_vp), ("M", c_vp), ("W", c_vp),
                ("valid", c_vp)]


class NvcScene(ctypes.Structure):
    _fields_ = [
        ("node_min", c_vp), ("node_max", c_vp),
        ("node_left", c_vp), ("node_right", c_vp), ("node_start", c_vp), ("node_count", c_vp),
        ("bv0", c_vp), ("bv1", c_vp), ("bv2", c_vp), ("perm", c_vp),
        ("tv0", c_vp), ("tv1", c_vp), ("tv2", c_vp),
        ("tri_material", c_vp), ("tri_light", c_vp), ("mat_albedo", c_vp),
        ("lt_kind", c_vp), ("lt_verts", c_vp), ("lt_normal", c_vp), ("lt_radiance", c_vp),
        ("lt_lumaw", c_vp), ("lt_area", c_vp),
        ("tri_plane", c_vp), ("tri_box", c_vp), ("tri_leaf", c_vp), ("node_parent", c_vp),
        ("plane_margin", ctypes.c_float), ("plane_r", ctypes.c_float), ("anyhit_bf", c_i32), ("pad0", c_i32),
        ("n_nodes", c_i64), ("n_tris", c_i64), ("n_lights", c_i32), ("n_materials", c_i32),
        ("shadow_eps", c_f64), ("aabb_min", c_f64 * 3), ("aabb_max", c_f64 * 3),
    ]


class NvcCamera(ctypes.Structure):
    _fields_ = [
        ("pos", c_f64 * 3), ("fwd", c_f64 * 3), ("right", c_f64 * 3), ("up", c_f64 * 3),
        ("tan_half", c_f64), ("aspect", c_f64), ("width", c_i32), ("height", c_i32),
    ]


P = ctypes.POINTER
_SIGS = {
    "nvc_last_error": (ctypes.c_char_p, []),
    "nvc_abi_version": (c_i32, []),
    "nvc_wpack_count": (c_i64, [P(NvcModel)]),
    "nvc_train_workspace_bytes": (c_i64, [P(NvcModel), c_i64]),
    "nvc_refresh_shadow": (c_i32, [P(NvcModel), c_vp]),
    "nvc_l2_persist": (c_i32, [c_vp, c_i64, c_vp]),
    "nvc_profile_stages": (c_i32, [c_i32]),
    "nvc_profile_stage_ms": (c_i32, [c_vp]),
    "nvc_encode": (c_i32, [P(NvcModel), c_vp, c_i64, c_vp, c_vp, c_vp, c_vp]),
    "nvc_infer": (c_i32, [P(NvcModel), c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "nvc_query_workspace_bytes": (c_i64, [P(NvcModel), c_i64]),
    "nvc_train_grads": (c_i32, [P(NvcModel), c_vp, c_vp, c_vp, c_i64, c_vp, c_i32, c_i32,
                                c_vp, c_vp, c_vp]),
    "nvc_adam_step": (c_i32, [P(NvcModel), c_i64, c_f64, c_vp]),
    "nvc_adam_step_shard": (c_i32, [P(NvcModel), c_i64, c_f64, c_i32, c_i32, c_vp]),
    "nvc_adam_shard_range": (c_i32, [P(NvcModel), c_i32, c_i32, P(c_i64), P(c_i64)]),
    "nvc_exchange_max_entries": (c_i64, [P(NvcModel), c_i64]),
    "nvc_touch_words": (c_i64, [P(NvcModel)]),
    "nvc_touch_off_len": (c_i64, [P(NvcModel)]),
    "nvc_train_index": (c_i32, [P(NvcModel), c_vp, c_i64, c_vp, c_vp]),
    "nvc_exchange_workspace_bytes": (c_i64, [P(NvcModel)]),
    "nvc_exchange_buffer_len": (c_i64, [P(NvcModel), c_i64]),
    "nvc_exchange_index": (c_i32, [P(NvcModel), c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "nvc_exchange_pack": (c_i32, [P(NvcModel), c_vp, c_vp, c_i64, c_vp, c_vp]),
    "nvc_exchange_unpack": (c_i32, [P(NvcModel), c_vp, c_vp, c_i64, c_vp, c_vp]),
    "nvc_wrs_select": (c_i32, [c_vp, c_i64, c_i32, c_u64, c_u64, c_vp, c_vp, c_vp, c_vp]),
    "nvc_nls_from_vis": (c_i32, [P(NvcScene), c_vp, c_vp, c_i32, c_i64, c_i64, c_i32, c_i64, c_i64,
                                 c_u64, c_u64, c_f64, c_vp, c_vp, c_vp, c_vp]),
    "nvc_nls_sample": (c_i32, [P(NvcModel), P(NvcScene), c_vp, c_vp, c_i32, c_vp, c_i64, c_i64, c_i64,
                               c_i64, c_u64, c_u64, c_f64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "nvc_query_front": (c_i32, [P(NvcModel), c_vp, c_i64, c_vp, c_vp]),
    "nvc_nls_select": (c_i32, [P(NvcModel), P(NvcScene), c_vp, c_i32, c_vp, c_i64, c_i64, c_i64, c_i64,
                               c_u64, c_u64, c_f64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "nvc_neural_di": (c_i32, [P(NvcModel), P(NvcScene), c_vp, c_vp, c_vp, c_i32, c_vp, c_i64, c_i64,
                              c_vp, c_vp, c_vp]),
    "nvc_table_mask": (c_i32, [c_vp, c_i32, c_i64, c_i64, c_i32, c_vp, c_vp]),
    "nvc_gbuffer": (c_i32, [P(NvcScene), P(NvcCamera), c_u64, c_i64, c_i64, c_vp, c_vp, c_vp,
                            c_vp, c_vp, c_vp, c_vp, c_vp]),
    "nvc_light_factors": (c_i32, [P(NvcScene), c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp,
                                  c_vp, c_vp]),
    "nvc_visibility": (c_i32, [P(NvcScene), c_vp, c_vp, c_i64, c_vp, c_vp]),
    "nvc_cluster_workspace_bytes": (c_i64, [c_i64, c_i32]),
    "nvc_cluster_state_offset": (c_i64, [c_i64, c_i32]),
    "nvc_cluster_targets": (c_i32, [P(NvcScene), c_u64, c_u64, c_i64, c_vp, c_vp, c_i64, c_i32, c_i32, c_i32, c_vp,
                                    c_vp, c_vp, c_vp, c_vp]),
    "nvc_clustered_workspace_bytes": (c_i64, [c_i64, c_i32]),
    "nvc_clustered_state_offset": (c_i64, [c_i64, c_i32]),
    "nvc_clustered_select": (c_i32, [P(NvcScene), c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_i32, c_vp, c_vp,
                                     c_u64, c_u64, c_f64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "nvc_cluster_factor_table": (c_i32, [c_vp, c_i64, c_i32, c_vp, c_vp, c_vp]),
    "nvc_clustered_select_ct": (c_i32, [P(NvcScene), c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i64, c_i64, c_i32, c_vp,
                                        c_vp, c_u64, c_u64, c_f64, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "nvc_shade": (c_i32, [P(NvcScene), c_vp, c_vp, c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "nvc_ris_workspace_bytes": (c_i64, [c_i64, c_i32, c_i32]),
    "nvc_ris_initial": (c_i32, [P(NvcScene), c_vp, c_i32, c_i64, c_i64, c_i32, c_u64, c_u64, c_i64,
                                P(NvcRGrid), c_vp, c_vp, c_vp]),
    "nvc_restir_temporal": (c_i32, [P(NvcScene), c_vp, c_i64, c_vp, c_i64, P(NvcRGrid), P(NvcRGrid), c_u64,
                                    c_u64, c_f64, c_i32, P(NvcRGrid), c_vp]),
    "nvc_restir_spatial": (c_i32, [P(NvcScene), c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_i32, c_i32,
                                   P(NvcRGrid), c_u64, c_u64, c_i32, c_i32, P(NvcRGrid), c_vp]),
    "nvc_phat_ids": (c_i32, [P(NvcScene), c_vp, c_i64, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "nvc_primary_hits": (c_i32, [P(NvcScene), P(NvcCamera), c_vp, c_i64, c_vp, c_vp, c_vp, c_vp, c_vp, c_vp]),
    "nvc_grid_scatter": (c_i32, [c_i32, c_i32, c_i64, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp]),
    "nvc_closest_hit": (c_i32, [P(NvcScene), c_vp, c_vp, c_vp, c_vp, c_i64, c_vp, c_vp, c_vp]),
    "nvc_batch_workspace_bytes": (c_i64, [c_i32, c_i32]),
    "nvc_targets": (c_i32, [P(NvcScene), c_u64, c_u64, c_vp, c_i64, c_vp, c_vp]),
    "nvc_gen_train_batch": (c_i32, [P(NvcScene), P(NvcCamera), c_u64, c_u64, c_u64, c_u64, c_u64, c_i32, c_i32,
                                    c_i32, c_i32, c_vp, c_vp, c_vp, c_vp, c_vp]),
}
EXPORTS = tuple(_SIGS)

_lib = None


class NvcError(RuntimeError):
    pass


class NvcUnsupported(NvcError):
    """A valid configuration the requested kernel does not cover (NVC_ERR_UNSUPPORTED)."""


def load_micro() -> ctypes.CDLL:
    """libnvc_micro.so (microbenchmarks; tools and bench rooflines only)."""
    p = os.path.join(os.path.dirname(LIB_PATH), "libnvc_micro.so")
    if not os.path.exists(p):
        raise ImportError(f"{p} is missing: python -m paper_2506_05930_b200.build")
    lib = ctypes.CDLL(p)
    c_vp, c_i32, c_i64, c_u32, c_u64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32, ctypes.c_uint64
    for name, args in {"nvc_micro": [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, c_vp, c_vp],
                       "nvc_encode_probe": [ctypes.POINTER(NvcModel), c_vp, c_i64, c_vp, c_vp],
                       "nvc_l2_gather_probe": [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp],
                       "nvc_philox_rate": [c_i32, c_i32, c_i32, c_u64, c_vp, c_vp],
                       "nvc_philox_check": [c_u64, c_u32, c_u32, c_vp, c_vp],
                       "nvc_l2_stream": [c_vp, c_i64, c_i32, c_i32, c_vp, c_vp]}.items():
        fn = getattr(lib, name)
        fn.restype = c_i32
        fn.argtypes = args
    return lib


def load(path: str | None = None) -> ctypes.CDLL:
    """Load libnvc.so (raises ImportError if it was never built)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise ImportError(f"{p} is missing: build it with `python -m paper_2506_05930_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(p)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if lib.nvc_abi_version() != ABI_VERSION:
        raise ImportError(f"libnvc ABI {lib.nvc_abi_version()} != {ABI_VERSION}")
    if path is None:
        _lib = lib
    return lib


def call(name: str, *args) -> None:
    lib = load()
    rc = getattr(lib, name)(*args)
    if rc != 0:
        msg = lib.nvc_last_error().decode(errors="replace")
        if rc == -1:
            raise ValueError(f"{name}: {msg}")
        if rc == -3:
            raise NvcUnsupported(f"{name}: {msg}")
        raise NvcError(f"{name} failed ({rc}): {msg}")


def ptr(t) -> int | None:
    """Raw device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(stream=None) -> int | None:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def require_cuda():
    import torch
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2506_05930_b200 needs a CUDA device (sm_100a); there is no CPU fallback")
    load()
    return torch


def f64_array(a, shape_tail=None) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape_tail is not None and a.shape[1:] != shape_tail:
        raise ValueError(f"expected shape (n,{','.join(map(str, shape_tail))}), got {a.shape}")
    return a
