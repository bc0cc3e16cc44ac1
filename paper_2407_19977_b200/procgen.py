"""Procedural test geometry -- the reference's procgen API (procgen.py:21-207):
an icosphere, a displaced sphere with an exact triangle count, and GLB
writers (`save_glb` lives with the ingest code, ingest.py).

The benchmark scenes (Cornell box, bunny-scale sphere, CAD pushbutton, HDR
sky) are workloads, not product API: see /workloads.py at the repo root.
"""
from __future__ import annotations

import math

import numpy as np

_PHI = (1.0 + math.sqrt(5.0)) / 2.0


def icosphere(subdivisions: int = 2, radius: float = 1.0) -> tuple[np.ndarray, np.ndarray]:
    """Subdivided icosahedron on a sphere (procgen.py:21-68): positions (n, 3)
    float64 and indices (3k,) int64, k = 20 * 4**subdivisions, watertight.
    Midpoints are created in face order, edge (a, b) once, so the vertex
    numbering is the reference's."""
    if subdivisions < 0:
        raise ValueError("subdivisions must be >= 0")
    if radius <= 0.0:
        raise ValueError("radius must be positive")
    p = _PHI
    base = np.array([[-1, p, 0], [1, p, 0], [-1, -p, 0], [1, -p, 0], [0, -1, p], [0, 1, p],
                     [0, -1, -p], [0, 1, -p], [p, 0, -1], [p, 0, 1], [-p, 0, -1], [-p, 0, 1]],
                    dtype=np.float64)
    verts = [v / np.linalg.norm(v) for v in base]
    faces = [(0, 11, 5), (0, 5, 1), (0, 1, 7), (0, 7, 10), (0, 10, 11), (1, 5, 9), (5, 11, 4),
             (11, 10, 2), (10, 7, 6), (7, 1, 8), (3, 9, 4), (3, 4, 2), (3, 2, 6), (3, 6, 8),
             (3, 8, 9), (4, 9, 5), (2, 4, 11), (6, 2, 10), (8, 6, 7), (9, 8, 1)]
    for _ in range(subdivisions):
        mids: dict[tuple[int, int], int] = {}

        def mid(a: int, b: int) -> int:
            key = (min(a, b), max(a, b))
            if key not in mids:
                m = verts[a] + verts[b]
                verts.append(m / np.linalg.norm(m))
                mids[key] = len(verts) - 1
            return mids[key]

        refined = []
        for a, b, c in faces:
            ab, bc, ca = mid(a, b), mid(b, c), mid(c, a)
            refined.extend([(a, ab, ca), (b, bc, ab), (c, ca, bc), (ab, bc, ca)])
        faces = refined
    return np.asarray(verts) * radius, np.asarray(faces, dtype=np.int64).ravel()


def bumpy_sphere(n_triangles: int, bump_amplitude: float = 0.12,
                 bump_frequencies=(6.0, 4.0), radius: float = 1.0):
    """Displaced lat/long sphere with exactly n_triangles faces; the same
    surface as the reference generator (procgen.py:71-114)."""
    if n_triangles < 1:
        raise ValueError("n_triangles must be >= 1")
    nu = max(int(math.ceil(math.sqrt(n_triangles / 2.0))), 1)
    nv = max(int(math.ceil(n_triangles / (2.0 * nu))), 1)
    fu, fv = bump_frequencies
    theta = np.linspace(math.pi / (nv + 2), math.pi * (nv + 1) / (nv + 2), nv + 1)
    phi = np.linspace(0.0, 2.0 * math.pi, nu + 1)
    tg, pg = np.meshgrid(theta, phi, indexing="ij")
    r = radius * (1.0 + bump_amplitude * np.sin(fu * tg) * np.cos(fv * pg))
    pos = np.stack([r * np.sin(tg) * np.cos(pg), r * np.cos(tg), r * np.sin(tg) * np.sin(pg)],
                   axis=-1).reshape(-1, 3)
    row = np.arange(nv)[:, None] * (nu + 1)
    col = np.arange(nu)[None, :]
    q00 = row + col
    q10 = q00 + (nu + 1)
    lower = np.stack([q00, q10, q00 + 1], axis=-1).reshape(-1, 3)
    upper = np.stack([q00 + 1, q10, q10 + 1], axis=-1).reshape(-1, 3)
    faces = np.empty((2 * lower.shape[0], 3), dtype=np.int64)
    faces[0::2], faces[1::2] = lower, upper
    return pos, faces[:n_triangles].ravel()



def icosphere_glb(path, subdivisions: int = 2, radius: float = 1.0,
                  material_name: str | None = None) -> int:
    """icosphere -> GLB with smooth normals (procgen.py:193-199); returns the
    triangle count."""
    from .ingest import generate_smooth_normals, save_glb
    positions, indices = icosphere(subdivisions, radius)
    save_glb(path, positions, indices, generate_smooth_normals(positions, indices), material_name)
    return indices.size // 3


def bumpy_sphere_glb(path, n_triangles: int, material_name: str | None = None) -> int:
    """bumpy_sphere -> GLB with smooth normals (procgen.py:202-207)."""
    from .ingest import generate_smooth_normals, save_glb
    positions, indices = bumpy_sphere(n_triangles)
    save_glb(path, positions, indices, generate_smooth_normals(positions, indices), material_name)
    return indices.size // 3
