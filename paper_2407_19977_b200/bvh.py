"""BVH types and closest-hit queries of the drop-in API (bvh.py of the
reference).

* `build_bvh` returns the reference's exact arrays from the GPU build
  (csrc/lt_bvh_gpu.cu) when a device is present, else from the host
  restatement (csrc/lt_bvh_build.cpp); a `DeviceScene` created without a BVH
  builds the same tree on the device without a host round trip.
* `intersect_scene_batch` / `intersect_scene` / `traversal_counts_batch`
  run the sm_100a traversal kernel through the C-ABI.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .geometry import Ray

LEAF_SIZE = 4          # bvh.py:22
SAH_BINS = 12          # bvh.py:23
MAX_TREE_DEPTH = 60    # bvh.py:26
STACK_SIZE = 64        # bvh.py:27


@dataclass
class BuildStats:
    node_count: int
    leaf_count: int
    max_depth: int
    build_time_ms: float


@dataclass
class Bvh:
    bounds_min: np.ndarray       # (node_count, 3) float64
    bounds_max: np.ndarray
    left_child: np.ndarray       # (node_count,) int32, -1 at leaves
    right_child: np.ndarray
    first_triangle: np.ndarray   # (node_count,) int32
    triangle_count: np.ndarray   # (node_count,) int32, 0 at internal nodes
    triangle_order: np.ndarray   # (n,) int32
    stats: BuildStats

    def is_leaf(self, node: int) -> bool:
        return self.triangle_count[node] > 0


GPU_MAX_BINS = 32


def build_bvh(triangles, leaf_size: int = LEAF_SIZE, bins: int = SAH_BINS, *,
              device="auto") -> Bvh:
    """Binned-SAH build (bvh.py:286-298); ValueError on an empty scene.

    Both builders return the reference's arrays: `device` = a CUDA ordinal
    runs csrc/lt_bvh_gpu.cu on that GPU; None runs the host restatement
    (csrc/lt_bvh_build.cpp); "auto" (default) uses GPU 0 when one is present
    and bins <= 32, else the host."""
    n = len(triangles)
    if n == 0:
        raise ValueError("empty scene")
    if device == "auto":
        device = 0 if bins <= GPU_MAX_BINS and _lib.device_count() > 0 else None
    v0 = np.ascontiguousarray(triangles.v0, dtype=np.float64)
    v1 = np.ascontiguousarray(triangles.v1, dtype=np.float64)
    v2 = np.ascontiguousarray(triangles.v2, dtype=np.float64)
    m = 2 * n
    bmin = np.empty((m, 3)); bmax = np.empty((m, 3))
    left = np.empty(m, np.int32); right = np.empty(m, np.int32)
    first = np.empty(m, np.int32); count = np.empty(m, np.int32)
    order = np.empty(n, np.int32)
    nn, nl, md = C.c_int64(), C.c_int64(), C.c_int64()
    P = _lib.ptr
    args = (P(v0, C.c_double), P(v1, C.c_double), P(v2, C.c_double), n, int(leaf_size),
            int(bins), P(bmin, C.c_double), P(bmax, C.c_double), P(left, C.c_int32),
            P(right, C.c_int32), P(first, C.c_int32), P(count, C.c_int32), P(order, C.c_int32),
            C.byref(nn), C.byref(nl), C.byref(md))
    t0 = time.perf_counter()
    if device is None:
        _lib.check(_lib.lib().lt_build_bvh(*args))
    else:
        _lib.check(_lib.lib().lt_build_bvh_device(int(device), *args))
    ms = (time.perf_counter() - t0) * 1e3
    k = int(nn.value)
    return Bvh(bmin[:k].copy(), bmax[:k].copy(), left[:k].copy(), right[:k].copy(),
               first[:k].copy(), count[:k].copy(), order,
               BuildStats(k, int(nl.value), int(md.value), ms))


def _rays(origins, directions):
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(directions, dtype=np.float64).reshape(-1, 3)
    if o.shape != d.shape:
        raise ValueError("origins and directions must have the same shape")
    return o, d


def intersect_scene_batch(triangles, bvh, origins, directions, t_min: float = 1e-4,
                          t_max: float = np.inf, *, device: int = 0, scene=None):
    """(indices int64, t float64) for many rays; -1 and +inf on a miss
    (bvh.py:667-677).  Traversal runs on the GPU in fp32; t is the fp32
    distance widened to float64.  Pass `scene` (a DeviceScene) to reuse a
    resident scene."""
    from .device import DeviceScene
    o, d = _rays(origins, directions)
    ds = scene if scene is not None else DeviceScene.from_geometry(triangles, bvh, device=device)
    idx = np.empty(o.shape[0], np.int64)
    t = np.empty(o.shape[0], np.float64)
    if o.shape[0]:
        P = _lib.ptr
        _lib.check(_lib.lib().lt_intersect_batch_host(
            ds.handle, P(o, C.c_double), P(d, C.c_double), o.shape[0], float(t_min),
            float(t_max), P(idx, C.c_int64), P(t, C.c_double)))
    return idx, t


def traversal_counts_batch(triangles, bvh, origins, directions, t_min: float = 1e-4,
                           t_max: float = np.inf, *, device: int = 0, scene=None):
    """(nodes_visited, triangle_tests) per ray from the GPU traversal
    (bvh.py:680-691)."""
    from .device import DeviceScene
    o, d = _rays(origins, directions)
    ds = scene if scene is not None else DeviceScene.from_geometry(triangles, bvh, device=device)
    nodes = np.empty(o.shape[0], np.int64)
    tests = np.empty(o.shape[0], np.int64)
    if o.shape[0]:
        P = _lib.ptr
        _lib.check(_lib.lib().lt_traversal_counts_host(
            ds.handle, P(o, C.c_double), P(d, C.c_double), o.shape[0], float(t_min),
            float(t_max), P(nodes, C.c_int64), P(tests, C.c_int64)))
    return nodes, tests


def intersect_any_batch(triangles, bvh, origins, directions, t_min: float = 1e-4,
                        t_max: float = np.inf, *, device: int = 0, scene=None) -> np.ndarray:
    """(n,) bool: any hit within [t_min, t_max] (the any-hit query of
    _traverse_any, bvh.py:511-551), on the GPU."""
    from .device import DeviceScene
    o, d = _rays(origins, directions)
    ds = scene if scene is not None else DeviceScene.from_geometry(triangles, bvh, device=device)
    out = np.zeros(o.shape[0], np.int32)
    if o.shape[0]:
        P = _lib.ptr
        _lib.check(_lib.lib().lt_occluded_batch_host(
            ds.handle, P(o, C.c_double), P(d, C.c_double), o.shape[0], float(t_min),
            float(t_max), P(out, C.c_int32)))
    return out.astype(bool)


def intersect_any(triangles, bvh, ray: Ray, *, device: int = 0, scene=None) -> bool:
    """intersect_any (bvh.py:658-664)."""
    return bool(intersect_any_batch(triangles, bvh, ray.origin[None], ray.direction[None],
                                    ray.t_min, ray.t_max, device=device, scene=scene)[0])


def intersect_scene(triangles, bvh, ray: Ray, *, device: int = 0, scene=None):
    """Nearest hit for one ray as (triangle_index, t) or None.  (The reference
    returns a Hit with normals; the hit frame is computed on the device inside
    the render kernels, so the scalar query reports index and distance.)"""
    idx, t = intersect_scene_batch(triangles, bvh, ray.origin[None], ray.direction[None],
                                   ray.t_min, ray.t_max, device=device, scene=scene)
    if idx[0] < 0:
        return None
    return int(idx[0]), float(t[0])
