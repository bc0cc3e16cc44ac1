"""The OpenPBR BSDF queries of the drop-in API (material.py:355-426 of the
reference) and the shade kernel's own BSDF code on explicit inputs.

* The public API -- `eval_bsdf` / `pdf_bsdf` / `sample_bsdf`, `ggx_ndf`,
  `smith_g2`, `cosine_sample_hemisphere`, `ggx_sample_half_vector` --
  runs the float64 device kernels of csrc/lt_query64.cu (the reference's
  arithmetic) for reference materials, so it returns the reference's
  numbers; materials with the coat / transmission extensions go through the
  shade kernel's code (fp32; no reference exists for them).
* `eval_pdf_batch` / `sample_batch` run the shade kernel's fp32 code
  (csrc/lt_material.cuh) through lt_bsdf_eval_ext_batch /
  lt_bsdf_sample_batch, so row a7 of the hot path is checked function by
  function against the reference (tests/test_gpu_functions.py).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib, query
from .material import EXTENSION_DEFAULTS


@dataclass(frozen=True)
class BsdfSample:
    direction: np.ndarray
    throughput_weight: np.ndarray   # f * cos(theta_i) / pdf
    pdf: float
    is_specular_spike: bool


def material_rows(materials) -> np.ndarray:
    """(n, 21) parameter rows (layout documented in include/luxb200.h)."""
    def g(m, name):
        return getattr(m, name, EXTENSION_DEFAULTS.get(name))
    rows = [[m.base_weight, *m.base_color, m.base_metalness, m.specular_weight,
             *m.specular_color, m.specular_roughness, m.specular_ior,
             g(m, "coat_weight"), g(m, "coat_roughness"), g(m, "coat_ior"), *g(m, "coat_color"),
             g(m, "transmission_weight"), *g(m, "transmission_color")] for m in materials]
    return np.ascontiguousarray(rows, dtype=np.float64).reshape(-1, 21)


def _v3(a, n):
    return np.ascontiguousarray(np.broadcast_to(np.asarray(a, dtype=np.float64), (n, 3)))


def eval_pdf_batch(params, wo, wi, normal, front=None):
    """(f (n,3), pdf (n,)) for n cases; `params` are OpenPbrParams-like
    objects or (n,21) rows.  For coat / transmission materials: the
    effective BSDF and density the extension sampler realizes (`front`: the
    geometric side, for the interface's eta; default outside)."""
    p = params if isinstance(params, np.ndarray) else material_rows(params)
    n = p.shape[0]
    wo, wi, nr = _v3(wo, n), _v3(wi, n), _v3(normal, n)
    fr = None if front is None else np.ascontiguousarray(
        np.broadcast_to(np.asarray(front, dtype=np.int32), (n,)))
    f = np.zeros((n, 3))
    pdf = np.zeros(n)
    P = _lib.ptr
    _lib.check(_lib.lib().lt_bsdf_eval_ext_batch(
        P(p, C.c_double), P(wo, C.c_double), P(wi, C.c_double), P(nr, C.c_double),
        P(fr, C.c_int32) if fr is not None else None, n, P(f, C.c_double),
        P(pdf, C.c_double)))
    return f, pdf


def sample_batch(params, wo, normal, draws, front=None):
    """(ok (n,), wi (n,3), weight (n,3)) for n cases with draws (n,3)."""
    p = params if isinstance(params, np.ndarray) else material_rows(params)
    n = p.shape[0]
    wo, nr = _v3(wo, n), _v3(normal, n)
    u = np.ascontiguousarray(np.asarray(draws, dtype=np.float64).reshape(n, 3))
    fr = None if front is None else np.ascontiguousarray(
        np.broadcast_to(np.asarray(front, dtype=np.int32), (n,)))
    ok = np.zeros(n, np.int32)
    wi = np.zeros((n, 3))
    w = np.zeros((n, 3))
    P = _lib.ptr
    _lib.check(_lib.lib().lt_bsdf_sample_batch(
        P(p, C.c_double), P(wo, C.c_double), P(nr, C.c_double), P(u, C.c_double),
        P(fr, C.c_int32) if fr is not None else None, n, P(ok, C.c_int32), P(wi, C.c_double),
        P(w, C.c_double)))
    return ok.astype(bool), wi, w


def _check_shading_frame(wo, n) -> None:
    """material.py:358-363."""
    if abs(float(np.linalg.norm(wo)) - 1.0) > 1e-6 or abs(float(np.linalg.norm(n)) - 1.0) > 1e-6:
        raise ValueError("wo and n must be unit length")
    if float(np.dot(wo, n)) <= 0.0:
        raise ValueError("wo must lie in the hemisphere of n")


def _extended(params) -> bool:
    return (float(getattr(params, "coat_weight", 0.0)) > 0.0
            or float(getattr(params, "transmission_weight", 0.0)) > 0.0)


def eval_bsdf(wo, wi, n, params) -> np.ndarray:
    """BSDF value (cosine excluded), material.py:389-398."""
    wo, wi, n = (np.asarray(x, dtype=np.float64) for x in (wo, wi, n))
    _check_shading_frame(wo, n)
    if _extended(params):
        return eval_pdf_batch([params], wo, wi, n)[0][0]
    return query.bsdf_eval_batch([params], wo, wi, n)[0][0]


def pdf_bsdf(wo, wi, n, params) -> float:
    """Solid-angle density of sample_bsdf, material.py:401-407."""
    wo, wi, n = (np.asarray(x, dtype=np.float64) for x in (wo, wi, n))
    _check_shading_frame(wo, n)
    if _extended(params):
        return float(eval_pdf_batch([params], wo, wi, n)[1][0])
    return float(query.bsdf_eval_batch([params], wo, wi, n)[1][0])


def sample_bsdf(wo, n, params, draws):
    """Importance sample with three unit draws (material.py:410-426); None
    for a zero-density outcome."""
    wo, n = np.asarray(wo, dtype=np.float64), np.asarray(n, dtype=np.float64)
    _check_shading_frame(wo, n)
    if _extended(params):
        ok, wi, w = sample_batch([params], wo, n, [draws])
        if not ok[0]:
            return None
        _, pdf = eval_pdf_batch([params], wo, wi, n)
        return BsdfSample(wi[0], w[0], float(pdf[0]), False)
    ok, wi, w, pdf, spike = query.bsdf_sample_batch([params], wo, n, [draws])
    if not ok[0]:
        return None
    return BsdfSample(wi[0], w[0], float(pdf[0]), bool(spike[0]))


def fresnel_schlick(cos_theta, f0, f90=1.0) -> np.ndarray:
    """material.py:366-369 (a host numpy expression in the reference too)."""
    f0 = np.asarray(f0, dtype=np.float64)
    f90 = np.asarray(f90, dtype=np.float64)
    return f0 + (f90 - f0) * (1.0 - cos_theta) ** 5


def ggx_ndf(n_dot_h: float, alpha: float) -> float:
    """material.py:372-373 (_ggx_ndf, 107-114), on the device in float64."""
    return float(query.microfacet(0, [float(n_dot_h)], [float(alpha)])[0])


def smith_g2(n_dot_o: float, n_dot_i: float, alpha: float) -> float:
    """material.py:376-377 (_smith_g2, 117-126), on the device in float64."""
    return float(query.microfacet(1, [float(n_dot_o)], [float(n_dot_i)], [float(alpha)])[0])


def cosine_sample_hemisphere(n, u1: float, u2: float) -> np.ndarray:
    """material.py:380-382 (_cosine_sample, 264-274)."""
    return query.microfacet(2, [float(u1)], [float(u2)], normal=[n])[0]


def ggx_sample_half_vector(n, alpha: float, u1: float, u2: float) -> np.ndarray:
    """material.py:385-387 (_ggx_sample_half, 277-290)."""
    return query.microfacet(3, [float(u1)], [float(u2)], [float(alpha)], normal=[n])[0]
