"""The reference's scalar query API, evaluated on the GPU in float64.

ray_triangle_intersect / ray_aabb_intersect (geometry.py:255-295), the hit
frame of intersect_scene (geometry.py:210-241), eval_bsdf / pdf_bsdf /
sample_bsdf and the microfacet helpers (material.py:366-426) and the
display transform (tonemap.py:18-61) run as batch kernels in
csrc/lt_query64.cu: float64 with the reference's operation order and no
FMA contraction, so these helpers return the reference's numbers.  (The
render path and the batch closest-hit queries are fp32; see integrator.py
and bvh.py.)  Every function here accepts batches; the scalar API wraps
them.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib

_d = C.c_double


def _f64(a, shape):
    return np.ascontiguousarray(np.broadcast_to(np.asarray(a, dtype=np.float64), shape))


def ray_triangle_batch(origins, dirs, t_min, t_max, v0, v1, v2, n0, n1, n2):
    """Per case one ray and one triangle: (ok (n,), tuv (n,3), geometric
    normal (n,3), shading normal (n,3), front (n,))."""
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    n = o.shape[0]
    d = _f64(dirs, (n, 3))
    lo, hi = _f64(t_min, (n,)), _f64(t_max, (n,))
    tri = [_f64(x, (n, 3)) for x in (v0, v1, v2, n0, n1, n2)]
    ok = np.zeros(n, np.int32)
    tuv, g, s = np.zeros((n, 3)), np.zeros((n, 3)), np.zeros((n, 3))
    front = np.zeros(n, np.int32)
    P = _lib.ptr
    _lib.check(_lib.lib().lt_ray_triangle_batch(P(o, _d), P(d, _d), P(lo, _d), P(hi, _d),
                                                *[P(x, _d) for x in tri], n, P(ok, C.c_int32),
                                                P(tuv, _d), P(g, _d), P(s, _d),
                                                P(front, C.c_int32)))
    return ok.astype(bool), tuv, g, s, front.astype(bool)


def hit_frame_batch(dirs, v0, v1, v2, n0, n1, n2, uv):
    """_hit_frame for each case: (geometric normal, shading normal, front)."""
    d = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
    n = d.shape[0]
    tri = [_f64(x, (n, 3)) for x in (v0, v1, v2, n0, n1, n2)]
    uvs = _f64(uv, (n, 2))
    g, s = np.zeros((n, 3)), np.zeros((n, 3))
    front = np.zeros(n, np.int32)
    P = _lib.ptr
    _lib.check(_lib.lib().lt_hit_frame_batch(P(d, _d), *[P(x, _d) for x in tri], P(uvs, _d), n,
                                             P(g, _d), P(s, _d), P(front, C.c_int32)))
    return g, s, front.astype(bool)


def ray_aabb_batch(origins, dirs, t_min, t_max, box_min, box_max):
    """(ok (n,), [t_enter, t_exit] (n,2))."""
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    n = o.shape[0]
    d = _f64(dirs, (n, 3))
    lo, hi = _f64(t_min, (n,)), _f64(t_max, (n,))
    bl, bh = _f64(box_min, (n, 3)), _f64(box_max, (n, 3))
    ok = np.zeros(n, np.int32)
    tnf = np.zeros((n, 2))
    P = _lib.ptr
    _lib.check(_lib.lib().lt_ray_aabb_batch(P(o, _d), P(d, _d), P(lo, _d), P(hi, _d), P(bl, _d),
                                            P(bh, _d), n, P(ok, C.c_int32), P(tnf, _d)))
    return ok.astype(bool), tnf


def material_params11(materials) -> np.ndarray:
    """(n, 11) reference material rows (material.py:68-92 order)."""
    rows = [[m.base_weight, *m.base_color, m.base_metalness, m.specular_weight,
             *m.specular_color, m.specular_roughness, m.specular_ior] for m in materials]
    return np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 11)


def bsdf_eval_batch(params, wo, wi, normal):
    """(f (n,3), pdf (n,)) of _eval_core / _pdf_core."""
    p = params if isinstance(params, np.ndarray) else material_params11(params)
    n = p.shape[0]
    a, b, c = _f64(wo, (n, 3)), _f64(wi, (n, 3)), _f64(normal, (n, 3))
    f, pdf = np.zeros((n, 3)), np.zeros(n)
    P = _lib.ptr
    _lib.check(_lib.lib().lt_bsdf64_eval_batch(P(p, _d), P(a, _d), P(b, _d), P(c, _d), n,
                                               P(f, _d), P(pdf, _d)))
    return f, pdf


def bsdf_sample_batch(params, wo, normal, draws):
    """(ok, wi, weight, pdf, spike) of _sample_core for each case."""
    p = params if isinstance(params, np.ndarray) else material_params11(params)
    n = p.shape[0]
    a, c = _f64(wo, (n, 3)), _f64(normal, (n, 3))
    u = _f64(draws, (n, 3))
    ok, spike = np.zeros(n, np.int32), np.zeros(n, np.int32)
    wi, w, pdf = np.zeros((n, 3)), np.zeros((n, 3)), np.zeros(n)
    P = _lib.ptr
    _lib.check(_lib.lib().lt_bsdf64_sample_batch(P(p, _d), P(a, _d), P(c, _d), P(u, _d), n,
                                                 P(ok, C.c_int32), P(wi, _d), P(w, _d),
                                                 P(pdf, _d), P(spike, C.c_int32)))
    return ok.astype(bool), wi, w, pdf, spike.astype(bool)


def microfacet(op: int, a, b, c=None, normal=None):
    """lt_microfacet_batch: 0 ggx_ndf, 1 smith_g2, 2 cosine sample, 3 GGX
    half vector (argument meaning in include/luxb200.h)."""
    a = np.atleast_1d(np.asarray(a, dtype=np.float64))
    n = a.shape[0]
    b = _f64(b, (n,))
    cc = _f64(c, (n,)) if c is not None else None
    nr = _f64(normal, (n, 3)) if normal is not None else None
    out = np.zeros((n, 3) if op >= 2 else n)
    P = _lib.ptr
    _lib.check(_lib.lib().lt_microfacet_batch(int(op), P(np.ascontiguousarray(a), _d), P(b, _d),
                                              P(cc, _d) if cc is not None else None,
                                              P(nr, _d) if nr is not None else None, n,
                                              P(out, _d)))
    return out


def display(op: int, values) -> np.ndarray:
    """lt_display_batch: 0 PBR Neutral over rgb triples, 1 linear -> sRGB,
    2 sRGB -> linear, 3 half-up u8 quantization; returns the input's shape."""
    x = np.ascontiguousarray(values, dtype=np.float64)
    flat = x.reshape(-1)
    n = flat.size // 3 if op == 0 else flat.size
    P = _lib.ptr
    if op == 3:
        out8 = np.zeros(flat.size, np.uint8)
        if n:
            _lib.check(_lib.lib().lt_display_batch(3, P(flat, _d), n, None, P(out8, C.c_uint8)))
        return out8.reshape(x.shape)
    out = np.zeros(flat.size)
    if n:
        _lib.check(_lib.lib().lt_display_batch(int(op), P(flat, _d), n, P(out, _d), None))
    return out.reshape(x.shape)
