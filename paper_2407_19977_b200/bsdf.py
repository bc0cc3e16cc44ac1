"""The OpenPBR BSDF of the shade kernel, callable on explicit inputs.

Mirrors luxtrace.material's query API (material.py:389-426: eval_bsdf,
pdf_bsdf, sample_bsdf) but runs the device code (csrc/lt_material.cuh) in
fp32 through lt_bsdf_eval_batch / lt_bsdf_sample_batch, so row a7 of the
hot path can be checked function by function against the reference.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _lib
from .material import EXTENSION_DEFAULTS


@dataclass(frozen=True)
class BsdfSample:
    direction: np.ndarray
    throughput_weight: np.ndarray   # f * cos(theta_i) / pdf


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


def eval_bsdf(wo, wi, n, params) -> np.ndarray:
    return eval_pdf_batch([params], wo, wi, n)[0][0]


def pdf_bsdf(wo, wi, n, params) -> float:
    return float(eval_pdf_batch([params], wo, wi, n)[1][0])


def sample_bsdf(wo, n, params, draws):
    ok, wi, w = sample_batch([params], wo, n, [draws])
    return BsdfSample(wi[0], w[0]) if ok[0] else None
