"""Geometry types and single-object queries of the drop-in API.

Mirrors luxtrace.geometry's public names (geometry.py:22-131, 255-315) so
callers can pass either these objects or the reference's own (duck-typed:
only the attributes are read).  The ray / triangle and ray / box queries
run the float64 device kernels of csrc/lt_query64.cu (the reference's
arithmetic); the AABB helpers are the reference's own numpy expressions.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

DET_EPSILON = 1e-9       # geometry.py:17
DEFAULT_T_MIN = 1e-4     # geometry.py:18
BOUNDS_PADDING = 1e-7    # geometry.py:19


def vec3(x: float, y: float, z: float) -> np.ndarray:
    return np.array([x, y, z], dtype=np.float64)


def normalize(v) -> np.ndarray:
    a = np.asarray(v, dtype=np.float64)
    length = float(np.linalg.norm(a))
    if length == 0.0:
        raise ValueError("cannot normalize zero vector")
    return a / length


@dataclass
class Ray:
    """A ray with unit direction and a closed interval [t_min, t_max]."""

    origin: np.ndarray
    direction: np.ndarray
    t_min: float = DEFAULT_T_MIN
    t_max: float = math.inf

    def __post_init__(self) -> None:
        self.origin = np.asarray(self.origin, dtype=np.float64)
        self.direction = np.asarray(self.direction, dtype=np.float64)
        if abs(float(np.linalg.norm(self.direction)) - 1.0) > 1e-6:
            raise ValueError("ray direction must be unit length")
        if not 0.0 <= self.t_min < self.t_max:
            raise ValueError(f"ray interval must satisfy 0 <= t_min < t_max, "
                             f"got [{self.t_min}, {self.t_max}]")


@dataclass
class Triangle:
    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray
    n0: np.ndarray
    n1: np.ndarray
    n2: np.ndarray
    material_index: int = 0


@dataclass
class Aabb:
    min: np.ndarray
    max: np.ndarray

    @classmethod
    def empty(cls) -> "Aabb":
        return cls(vec3(math.inf, math.inf, math.inf), vec3(-math.inf, -math.inf, -math.inf))

    def is_empty(self) -> bool:
        return bool(np.any(self.min > self.max))


@dataclass
class Hit:
    t: float
    triangle_index: int
    barycentric_u: float
    barycentric_v: float
    geometric_normal: np.ndarray
    shading_normal: np.ndarray
    is_front_face: bool


_CORNERS = ("v0", "v1", "v2", "n0", "n1", "n2")


@dataclass
class TriangleBuffer:
    """Structure-of-arrays triangle soup: six (n, 3) float64 arrays and an
    (n,) int32 material index, the layout the reference packs for its
    kernels (geometry.py:88-131)."""

    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray
    n0: np.ndarray
    n1: np.ndarray
    n2: np.ndarray
    material_index: np.ndarray = field(default=None)

    def __post_init__(self) -> None:
        for name in _CORNERS:
            a = np.ascontiguousarray(getattr(self, name), dtype=np.float64)
            if a.ndim != 2 or a.shape[1] != 3:
                raise ValueError(f"{name} must have shape (n, 3), got {a.shape}")
            setattr(self, name, a)
        n = self.v0.shape[0]
        if any(getattr(self, k).shape[0] != n for k in _CORNERS):
            raise ValueError("all corner arrays must have the same length")
        mi = np.zeros(n, np.int32) if self.material_index is None else self.material_index
        self.material_index = np.ascontiguousarray(mi, dtype=np.int32)
        if self.material_index.shape != (n,):
            raise ValueError("material_index must have shape (n,)")

    def __len__(self) -> int:
        return int(self.v0.shape[0])

    def __getitem__(self, i: int) -> Triangle:
        return Triangle(*(getattr(self, k)[i].copy() for k in _CORNERS),
                        int(self.material_index[i]))

    @classmethod
    def from_triangles(cls, triangles) -> "TriangleBuffer":
        tris = list(triangles)
        cols = {k: np.array([getattr(t, k) for t in tris], dtype=np.float64) for k in _CORNERS}
        return cls(**cols, material_index=np.array([t.material_index for t in tris], np.int32))


# ------------------------------------------------------------------ queries

def ray_triangle_intersect(ray: Ray, tri: Triangle, triangle_index: int = 0) -> Hit | None:
    """Nearest double-sided hit of one ray with one triangle (geometry.py:
    255-278): _mt_intersect + _hit_frame in float64 on the device."""
    from . import query
    ok, tuv, g, s, front = query.ray_triangle_batch(
        ray.origin, ray.direction, ray.t_min, ray.t_max, tri.v0, tri.v1, tri.v2, tri.n0, tri.n1,
        tri.n2)
    if not ok[0]:
        return None
    t, u, v = tuv[0]
    return Hit(float(t), triangle_index, float(u), float(v), g[0].copy(), s[0].copy(),
               bool(front[0]))


def ray_aabb_intersect(ray: Ray, box: Aabb):
    """Clipped slab interval (t_enter, t_exit) or None (geometry.py:281-295),
    the reference's NaN-tolerant compare / select form, float64 on the
    device."""
    from . import query
    ok, tnf = query.ray_aabb_batch(ray.origin, ray.direction, ray.t_min, ray.t_max, box.min,
                                   box.max)
    if not ok[0]:
        return None
    return float(tnf[0, 0]), float(tnf[0, 1])


def triangle_bounds(tri: Triangle) -> Aabb:
    """AABB of a triangle padded by BOUNDS_PADDING times its max extent
    (geometry.py:298-304)."""
    lo = np.minimum(np.minimum(tri.v0, tri.v1), tri.v2)
    hi = np.maximum(np.maximum(tri.v0, tri.v1), tri.v2)
    pad = BOUNDS_PADDING * float(np.max(hi - lo))
    return Aabb(lo - pad, hi + pad)


def aabb_union(a: Aabb, b: Aabb) -> Aabb:
    return Aabb(np.minimum(a.min, b.min), np.maximum(a.max, b.max))


def aabb_surface_area(box: Aabb) -> float:
    if box.is_empty():
        return 0.0
    d = box.max - box.min
    return float(2.0 * (d[0] * d[1] + d[0] * d[2] + d[1] * d[2]))
