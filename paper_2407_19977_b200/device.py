"""Device-resident scene: the lt_scene handle behind every GPU call.

`DeviceScene(scene, bvh)` packs the same arrays the reference's
`_scene_arrays` (integrator.py:284-291) hands to `_render_pass` and uploads
them once through lt_scene_create, which flattens the host BVH into the fp32
HBM layout on the device.  Reference objects (luxtrace SceneDescription /
TriangleBuffer / Bvh / OpenPbrParams) are accepted duck-typed.
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np

from . import _lib
from .material import pack_material_table
from .scene import environment_pack


def _c64(a, shape=None) -> np.ndarray:
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and out.shape != shape:
        out = out.reshape(shape)
    return out


def _c32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int32)


def _shading_desc(d, materials, environment, keep) -> int:
    """Material table + environment fields of an lt_scene_desc; returns the
    material count."""
    def p64(a):
        arr = _c64(a)
        keep.append(arr)
        return arr.ctypes.data_as(C.POINTER(C.c_double))

    table = pack_material_table(materials)
    d.n_materials = len(table["base_weight"])
    for name, arr in table.items():
        setattr(d, name, p64(arr))
    kind, a, b = environment_pack(environment)
    d.env_kind = kind
    d.env_a[:] = [float(x) for x in a]
    d.env_b[:] = [float(x) for x in b]
    if kind == _lib.LT_ENV_LATLONG:
        tex = np.ascontiguousarray(environment.texels, dtype=np.float32)
        keep.append(tex)
        d.env_height, d.env_width = int(tex.shape[0]), int(tex.shape[1])
        d.env_texels = tex.ctypes.data_as(C.POINTER(C.c_float))
        d.env_scale = float(environment.scale)
    return d.n_materials


class DeviceScene:
    """Owns one lt_scene on one GPU.  Not thread-safe; one per device."""

    def __init__(self, scene, bvh=None, device: int = 0):
        self._init(scene.triangles, bvh, scene.materials, scene.environment, device)
        self.camera = scene.camera

    @classmethod
    def from_geometry(cls, triangles, bvh=None, materials=None, environment=None,
                      device: int = 0) -> "DeviceScene":
        from .material import OpenPbrParams
        from .scene import EnvironmentConfig
        self = cls.__new__(cls)
        n_mat = int(np.max(triangles.material_index)) + 1 if len(triangles) else 1
        self._init(triangles, bvh, materials or [OpenPbrParams()] * n_mat,
                   environment or EnvironmentConfig.uniform((0.0, 0.0, 0.0)), device)
        self.camera = None
        return self

    def _init(self, triangles, bvh, materials, environment, device):
        _lib.require_gpu()
        self.handle = None
        # bvh None: lt_scene_create builds the reference's tree on the device
        # (no host round trip); `self.bvh` stays None
        self.bvh = bvh
        n = len(triangles)
        keep = []  # arrays must stay alive until lt_scene_create returns

        def p64(a, shape=None):
            arr = _c64(a, shape)
            keep.append(arr)
            return arr.ctypes.data_as(C.POINTER(C.c_double))

        def p32(a):
            arr = _c32(a)
            keep.append(arr)
            return arr.ctypes.data_as(C.POINTER(C.c_int32))

        d = _lib.SceneDesc()
        d.n_triangles = n
        d.v0, d.v1, d.v2 = (p64(triangles.v0), p64(triangles.v1), p64(triangles.v2))
        d.n0, d.n1, d.n2 = (p64(triangles.n0), p64(triangles.n1), p64(triangles.n2))
        d.material_index = p32(triangles.material_index)
        if bvh is None:
            d.n_nodes = 0       # all BVH pointers stay NULL
        else:
            nn = int(np.asarray(bvh.left_child).shape[0])
            d.n_nodes = nn
            d.bounds_min = p64(bvh.bounds_min, (nn, 3))
            d.bounds_max = p64(bvh.bounds_max, (nn, 3))
            d.left_child, d.right_child = p32(bvh.left_child), p32(bvh.right_child)
            d.first_triangle = p32(bvh.first_triangle)
            d.triangle_count = p32(bvh.triangle_count)
            d.triangle_order = p32(bvh.triangle_order)
        self.n_materials = _shading_desc(d, materials, environment, keep)
        handle = C.c_void_p()
        t0 = time.perf_counter()
        _lib.check(_lib.lib().lt_scene_create(C.byref(d), int(device), C.byref(handle)))
        self.create_ms = (time.perf_counter() - t0) * 1e3
        self._adopt(handle, device, n)

    @classmethod
    def from_gltf(cls, gltf, keep, materials, environment, camera, device: int = 0):
        """Scene from a glTF description (`_lib.GltfDesc`, whose arrays `keep`
        holds alive) flattened on the device by lt_scene_create_gltf: the
        triangle soup never exists on the host.  Sets `degenerate_dropped`."""
        _lib.require_gpu()
        self = cls.__new__(cls)
        self.handle = None
        self.bvh = None
        d = _lib.SceneDesc()
        keep = list(keep)
        self.n_materials = _shading_desc(d, materials, environment, keep)
        handle = C.c_void_p()
        kept, dropped = C.c_int64(0), C.c_int64(0)
        t0 = time.perf_counter()
        _lib.check(_lib.lib().lt_scene_create_gltf(C.byref(gltf), C.byref(d), int(device),
                                                   C.byref(handle), C.byref(kept),
                                                   C.byref(dropped)))
        self.create_ms = (time.perf_counter() - t0) * 1e3
        self._adopt(handle, device, kept.value)
        self.degenerate_dropped = dropped.value
        self.camera = camera
        return self

    def _adopt(self, handle, device, n) -> None:
        self.handle = handle
        self.device = int(device)
        self.n_triangles = n
        info = _lib.SceneInfo()
        _lib.check(_lib.lib().lt_scene_info_get(handle, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in info._fields_}

    def close(self) -> None:
        if getattr(self, "handle", None):
            _lib.lib().lt_scene_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def stats(self) -> dict:
        s = _lib.RenderStats()
        _lib.check(_lib.lib().lt_render_stats_get(self.handle, C.byref(s)))
        return {f: getattr(s, f) for f, _ in s._fields_}
