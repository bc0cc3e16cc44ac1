"""BVH types and closest-hit queries of the drop-in API (bvh.py of the
reference).

* `build_bvh` returns the reference's exact arrays from the GPU build
  (csrc/lt_bvh_gpu.cu) when a device is present, else from the host
  restatement (csrc/lt_bvh_build.cpp); a `DeviceScene` created without a BVH
  builds the same tree on the device without a host round trip.
* `intersect_scene_batch` / `intersect_scene` / `intersect_scene_counted` /
  `traversal_counts_batch` run the sm_100a traversal kernel through the
  C-ABI (fp32); `intersect_scene` builds the reference's `Hit` with the
  float64 hit frame on the device; `brute_force_intersect_batch` is the
  exhaustive GPU kernel with the traversal's arithmetic, so the two agree
  exactly (test_bvh.py:91-100);
* `validate_bvh` is the reference's structural checker (bvh.py:305-352),
  host numpy over the tree arrays.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass

import numpy as np

from . import _lib
from .geometry import BOUNDS_PADDING, Hit, Ray

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


def intersect_hits_batch(triangles, bvh, origins, directions, t_min: float = 1e-4,
                         t_max: float = np.inf, *, device: int = 0, scene=None):
    """(indices, t, uv (n,2)) of the fp32 traversal."""
    from .device import DeviceScene
    o, d = _rays(origins, directions)
    ds = scene if scene is not None else DeviceScene.from_geometry(triangles, bvh, device=device)
    idx = np.empty(o.shape[0], np.int64)
    t = np.empty(o.shape[0], np.float64)
    uv = np.zeros((o.shape[0], 2), np.float64)
    if o.shape[0]:
        P = _lib.ptr
        _lib.check(_lib.lib().lt_intersect_hits_host(
            ds.handle, P(o, C.c_double), P(d, C.c_double), o.shape[0], float(t_min),
            float(t_max), P(idx, C.c_int64), P(t, C.c_double), P(uv, C.c_double)))
    return idx, t, uv


def _hit(triangles, ray: Ray, k: int, t: float, uv) -> Hit:
    """_hit_from_traverse (bvh.py:617-629): the float64 hit frame of
    triangle k at the traversal's (u, v), on the device."""
    from . import query
    g, s, front = query.hit_frame_batch(ray.direction, triangles.v0[k], triangles.v1[k],
                                        triangles.v2[k], triangles.n0[k], triangles.n1[k],
                                        triangles.n2[k], uv)
    return Hit(float(t), int(k), float(uv[0]), float(uv[1]), g[0], s[0], bool(front[0]))


def intersect_scene(triangles, bvh, ray: Ray, *, device: int = 0, scene=None):
    """Nearest hit of one ray as the reference's Hit, or None (bvh.py:
    632-641)."""
    idx, t, uv = intersect_hits_batch(triangles, bvh, ray.origin[None], ray.direction[None],
                                      ray.t_min, ray.t_max, device=device, scene=scene)
    if idx[0] < 0:
        return None
    return _hit(triangles, ray, int(idx[0]), t[0], uv[0])


def intersect_scene_counted(triangles, bvh, ray: Ray, *, device: int = 0, scene=None):
    """(hit, nodes_visited, triangle_tests), bvh.py:644-655: the hit of the
    render traversal and the work counters of the reference-order binary
    traversal (traversal_counts_batch)."""
    from .device import DeviceScene
    ds = scene if scene is not None else DeviceScene.from_geometry(triangles, bvh, device=device)
    hit = intersect_scene(triangles, bvh, ray, scene=ds)
    nodes, tests = traversal_counts_batch(triangles, bvh, ray.origin[None], ray.direction[None],
                                          ray.t_min, ray.t_max, scene=ds)
    return hit, int(nodes[0]), int(tests[0])


def brute_force_intersect_batch(triangles, origins, directions, t_min: float = 1e-4,
                                t_max: float = np.inf, *, device: int = 0, scene=None):
    """(indices, t) by testing every triangle (bvh.py:694-701), on the GPU
    with the traversal's fp32 Moller-Trumbore and tie rule."""
    from .device import DeviceScene
    o, d = _rays(origins, directions)
    ds = scene if scene is not None else DeviceScene.from_geometry(triangles, None, device=device)
    idx = np.empty(o.shape[0], np.int64)
    t = np.empty(o.shape[0], np.float64)
    if o.shape[0]:
        P = _lib.ptr
        _lib.check(_lib.lib().lt_brute_force_batch_host(
            ds.handle, P(o, C.c_double), P(d, C.c_double), o.shape[0], float(t_min),
            float(t_max), P(idx, C.c_int64), P(t, C.c_double)))
    return idx, t


def triangle_bounds_arrays(v0, v1, v2):
    """_triangle_bounds_arrays (bvh.py:57-77): padded per-triangle boxes and
    centroids, the same float64 operations."""
    lo = np.minimum(v0, np.minimum(v1, v2))
    hi = np.maximum(v0, np.maximum(v1, v2))
    ext = np.maximum((hi - lo).max(axis=1), 0.0)
    pad = (BOUNDS_PADDING * ext)[:, None]
    lo = lo - pad
    hi = hi + pad
    return lo, hi, 0.5 * (lo + hi)


def validate_bvh(bvh, triangles, tolerance: float = 1e-6) -> list[str]:
    """Structural checks of a tree (bvh.py:305-352); returns the violations
    in the reference's wording (empty = valid)."""
    out: list[str] = []
    n_nodes = bvh.bounds_min.shape[0]
    n = len(triangles)
    leaf = bvh.triangle_count > 0
    internal = ~leaf
    idx = np.arange(n_nodes)
    for name, child in (("left", bvh.left_child), ("right", bvh.right_child)):
        for i in np.nonzero(internal & (child <= idx))[0]:
            out.append(f"node {i}: {name} child {child[i]} does not have a larger index")
        for i in np.nonzero(internal & (child < 0))[0]:
            out.append(f"node {i}: internal node lacks a {name} child")
    ok_children = internal & (bvh.left_child > idx) & (bvh.right_child > idx)
    for i in np.nonzero(ok_children)[0]:
        for ci in (bvh.left_child[i], bvh.right_child[i]):
            if np.any(bvh.bounds_min[ci] < bvh.bounds_min[i] - tolerance) or \
               np.any(bvh.bounds_max[ci] > bvh.bounds_max[i] + tolerance):
                out.append(f"node {i}: child {ci} bounds exceed parent bounds")
    if sorted(np.asarray(bvh.triangle_order).tolist()) != list(range(n)):
        out.append("triangle_order is not a permutation of [0, n)")
    tb_min, tb_max, _ = triangle_bounds_arrays(np.asarray(triangles.v0, np.float64),
                                               np.asarray(triangles.v1, np.float64),
                                               np.asarray(triangles.v2, np.float64))
    covered = np.zeros(n, dtype=np.int64)
    for i in np.nonzero(leaf)[0]:
        f = int(bvh.first_triangle[i])
        c = int(bvh.triangle_count[i])
        if c < 1:
            out.append(f"node {i}: leaf with no triangles")
            continue
        if f < 0 or f + c > n:
            out.append(f"node {i}: leaf range [{f}, {f + c}) out of bounds")
            continue
        members = bvh.triangle_order[f:f + c]
        covered[members] += 1
        if np.any(tb_min[members] < bvh.bounds_min[i] - tolerance) or \
           np.any(tb_max[members] > bvh.bounds_max[i] + tolerance):
            out.append(f"node {i}: leaf bounds do not contain member triangle bounds")
    if np.any(covered != 1):
        bad = np.nonzero(covered != 1)[0]
        out.append(f"triangles not covered by exactly one leaf: {bad[:8].tolist()}"
                   + ("..." if bad.size > 8 else ""))
    return out
