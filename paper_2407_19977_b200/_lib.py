"""ctypes binding of the C-ABI in include/luxb200.h.

The product path has no CPU fallback: if libluxb200.so is missing or no CUDA
device is present, every compute entry point raises.  Struct layouts mirror
the header field for field (ctypes applies the same C alignment rules).
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("LUXB200_LIB",
                               Path(__file__).resolve().parent / "_build" / "libluxb200.so"))

LT_OK = 0
LT_ERR_INVALID = 1
LT_ERR_CUDA = 2
LT_ERR_NOMEM = 3
LT_ERR_UNSUPPORTED = 4

LT_ENV_UNIFORM = 0
LT_ENV_GRADIENT = 1
LT_ENV_LATLONG = 2

LT_FLAG_SORT_MATERIALS = 1
LT_FLAG_PROFILE = 4
LT_FLAG_COUNT = 8

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_up = C.POINTER(C.c_uint64)
_u32p = C.POINTER(C.c_uint32)
_u8p = C.POINTER(C.c_uint8)


class SceneDesc(C.Structure):
    _fields_ = [
        ("n_triangles", C.c_int64),
        ("v0", _dp), ("v1", _dp), ("v2", _dp), ("n0", _dp), ("n1", _dp), ("n2", _dp),
        ("material_index", _ip),
        ("n_nodes", C.c_int64),
        ("bounds_min", _dp), ("bounds_max", _dp),
        ("left_child", _ip), ("right_child", _ip),
        ("first_triangle", _ip), ("triangle_count", _ip),
        ("triangle_order", _ip),
        ("n_materials", C.c_int32),
        ("base_weight", _dp), ("base_color", _dp), ("base_metalness", _dp),
        ("specular_weight", _dp), ("specular_color", _dp), ("specular_roughness", _dp),
        ("specular_ior", _dp), ("emission_luminance", _dp), ("emission_color", _dp),
        ("coat_weight", _dp), ("coat_roughness", _dp), ("coat_ior", _dp), ("coat_color", _dp),
        ("transmission_weight", _dp), ("transmission_color", _dp),
        ("env_kind", C.c_int32),
        ("env_a", C.c_double * 3), ("env_b", C.c_double * 3),
        ("env_width", C.c_int32), ("env_height", C.c_int32),
        ("env_texels", _fp),
        ("env_scale", C.c_double),
    ]


class SceneInfo(C.Structure):
    _fields_ = [
        ("device", C.c_int32),
        ("n_triangles", C.c_int64), ("n_nodes", C.c_int64), ("n_internal", C.c_int64),
        ("device_bytes", C.c_int64),
        ("sm_count", C.c_int32),
        ("n_wide", C.c_int64), ("l2_persist_bytes", C.c_int64), ("l2_window_bytes", C.c_int64),
        ("default_batch_paths", C.c_int64),
    ]


class RenderParams(C.Structure):
    _fields_ = [
        ("camera", C.c_double * 14),
        ("width", C.c_int32), ("height", C.c_int32),
        ("sample_start", C.c_int64), ("sample_count", C.c_int64),
        ("seed", C.c_uint64),
        ("max_depth", C.c_int32), ("rr_start", C.c_int32),
        ("t_min", C.c_double),
        ("tile_size", C.c_int32), ("rank", C.c_int32), ("n_ranks", C.c_int32),
        ("flags", C.c_uint32),
        ("max_batch_paths", C.c_int64),
    ]


class RenderStats(C.Structure):
    _fields_ = [
        ("paths", C.c_int64), ("rays", C.c_int64), ("batches", C.c_int64),
        ("kernel_launches", C.c_int64), ("trace_launches", C.c_int64),
        ("slab_tests", C.c_int64), ("tri_tests", C.c_int64),
        ("trace_ms", C.c_double),
        ("shade_warps", C.c_int64), ("shade_mixed_warps", C.c_int64),
        ("shade_warp_classes", C.c_int64),
    ]


class GltfPrimitive(C.Structure):
    _fields_ = [
        ("pos_buffer", C.c_int32), ("pos_stride", C.c_int32),
        ("pos_offset", C.c_int64), ("n_vertices", C.c_int64),
        ("nrm_buffer", C.c_int32), ("nrm_stride", C.c_int32),
        ("nrm_offset", C.c_int64),
        ("idx_buffer", C.c_int32), ("idx_stride", C.c_int32), ("idx_bytes", C.c_int32),
        ("reserved", C.c_int32),
        ("idx_offset", C.c_int64), ("n_indices", C.c_int64),
    ]


class GltfInstance(C.Structure):
    _fields_ = [
        ("primitive", C.c_int32), ("material", C.c_int32),
        ("linear", C.c_double * 9), ("translation", C.c_double * 3),
        ("normal_matrix", C.c_double * 9),
    ]


class GltfDesc(C.Structure):
    _fields_ = [
        ("n_buffers", C.c_int32), ("buffers", C.POINTER(_u8p)), ("buffer_bytes", _lp),
        ("n_primitives", C.c_int32), ("primitives", C.POINTER(GltfPrimitive)),
        ("n_instances", C.c_int32), ("instances", C.POINTER(GltfInstance)),
    ]


# (name, restype, argtypes) for every symbol the header declares
SIGNATURES = {
    "lt_abi_version": (C.c_int, []),
    "lt_last_error": (C.c_char_p, []),
    "lt_device_count": (C.c_int, [_ip]),
    "lt_build_bvh": (C.c_int, [_dp, _dp, _dp, C.c_int64, C.c_int32, C.c_int32, _dp, _dp, _ip,
                               _ip, _ip, _ip, _ip, _lp, _lp, _lp]),
    "lt_build_bvh_device": (C.c_int, [C.c_int32, _dp, _dp, _dp, C.c_int64, C.c_int32, C.c_int32,
                                      _dp, _dp, _ip, _ip, _ip, _ip, _ip, _lp, _lp, _lp]),
    "lt_scene_create": (C.c_int, [C.POINTER(SceneDesc), C.c_int32, C.POINTER(C.c_void_p)]),
    "lt_scene_create_gltf": (C.c_int, [C.POINTER(GltfDesc), C.POINTER(SceneDesc), C.c_int32,
                                       C.POINTER(C.c_void_p), _lp, _lp]),
    "lt_gltf_flatten": (C.c_int, [C.POINTER(GltfDesc), C.c_int32, C.c_int64, _dp, _dp, _dp, _dp,
                                  _dp, _dp, _ip, _lp, _lp]),
    "lt_scene_destroy": (C.c_int, [C.c_void_p]),
    "lt_scene_info_get": (C.c_int, [C.c_void_p, C.POINTER(SceneInfo)]),
    "lt_intersect_batch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_float,
                                     C.c_float, C.c_void_p, C.c_void_p, C.c_void_p]),
    "lt_intersect_batch_host": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int64, C.c_double,
                                          C.c_double, _lp, _dp]),
    "lt_intersect_hits_host": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int64, C.c_double,
                                         C.c_double, _lp, _dp, _dp]),
    "lt_brute_force_batch_host": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int64, C.c_double,
                                            C.c_double, _lp, _dp]),
    "lt_ray_triangle_batch": (C.c_int, [_dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp,
                                        C.c_int64, _ip, _dp, _dp, _dp, _ip]),
    "lt_hit_frame_batch": (C.c_int, [_dp, _dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_int64, _dp,
                                     _dp, _ip]),
    "lt_ray_aabb_batch": (C.c_int, [_dp, _dp, _dp, _dp, _dp, _dp, C.c_int64, _ip, _dp]),
    "lt_bsdf64_eval_batch": (C.c_int, [_dp, _dp, _dp, _dp, C.c_int64, _dp, _dp]),
    "lt_bsdf64_sample_batch": (C.c_int, [_dp, _dp, _dp, _dp, C.c_int64, _ip, _dp, _dp, _dp,
                                         _ip]),
    "lt_microfacet_batch": (C.c_int, [C.c_int32, _dp, _dp, _dp, _dp, C.c_int64, _dp]),
    "lt_display_batch": (C.c_int, [C.c_int32, _dp, C.c_int64, _dp, _u8p]),
    "lt_traversal_counts_host": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int64, C.c_double,
                                           C.c_double, _lp, _lp]),
    "lt_render_pass": (C.c_int, [C.c_void_p, C.POINTER(RenderParams), C.c_void_p, C.c_void_p,
                                 C.c_void_p, C.c_void_p]),
    "lt_render_pass_host": (C.c_int, [C.c_void_p, C.POINTER(RenderParams), _dp, _lp, _lp]),
    "lt_render_stats_get": (C.c_int, [C.c_void_p, C.POINTER(RenderStats)]),
    "lt_trace_paths_host": (C.c_int, [C.c_void_p, _dp, _dp, _up, _up, C.c_int64, C.c_int32,
                                      C.c_int32, C.c_double, _dp, _up]),
    "lt_tonemap_u8": (C.c_int, [C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p]),
    "lt_accum_finish": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p,
                                  C.c_void_p, C.c_void_p]),
    "lt_read_bandwidth": (C.c_int, [C.c_int32, C.c_int64, C.c_int32, C.POINTER(C.c_double)]),
    "lt_bsdf_eval_batch": (C.c_int, [_dp, _dp, _dp, _dp, C.c_int64, _dp, _dp]),
    "lt_bsdf_eval_ext_batch": (C.c_int, [_dp, _dp, _dp, _dp, _ip, C.c_int64, _dp, _dp]),
    "lt_bsdf_sample_batch": (C.c_int, [_dp, _dp, _dp, _dp, _ip, C.c_int64, _ip, _dp, _dp]),
    "lt_occluded_batch_host": (C.c_int, [C.c_void_p, _dp, _dp, C.c_int64, C.c_double,
                                         C.c_double, _ip]),
}


def read_bandwidth(device: int, nbytes: int, iters: int = 20) -> float:
    """GB/s of a streaming read over an `nbytes` device buffer."""
    g = C.c_double()
    check(lib().lt_read_bandwidth(int(device), int(nbytes), int(iters), C.byref(g)))
    return float(g.value)

_lib = None


class NativeLibraryMissing(RuntimeError):
    pass


def lib():
    """The loaded libluxb200.so (built in-tree by build.py); raises if absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise NativeLibraryMissing(
            f"{LIB_PATH} is missing: run `python -m paper_2407_19977_b200.build` "
            "(there is no CPU fallback)")
    handle = C.CDLL(str(LIB_PATH))
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.lt_abi_version() != 2:
        raise NativeLibraryMissing("libluxb200.so ABI version mismatch")
    _lib = handle
    return _lib


def check(rc: int) -> None:
    if rc == LT_OK:
        return
    msg = lib().lt_last_error().decode(errors="replace")
    if rc == LT_ERR_INVALID:
        raise ValueError(msg)
    if rc == LT_ERR_NOMEM:
        raise MemoryError(msg)
    raise RuntimeError(f"luxb200 error {rc}: {msg}")


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


def device_count() -> int:
    n = C.c_int32(0)
    rc = lib().lt_device_count(C.byref(n))
    return int(n.value) if rc == LT_OK else 0


def require_gpu() -> None:
    if device_count() < 1:
        raise RuntimeError("luxb200 needs a CUDA device (B200, sm_100a); no CPU fallback")


if os.environ.get("LUXB200_EAGER_LOAD"):
    lib()
