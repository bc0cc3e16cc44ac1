"""OpenPBR-subset material parameters (material.py:25-92 of the reference),
extended with the coat and transmission lobes the north star adds.

The extension fields default to zero weight, and a zero-weight material is
the reference material bit for bit: the kernels skip the extension chain
entirely (see csrc/lt_material.cuh).  Reference `OpenPbrParams` objects are
accepted as-is; missing extension attributes read as their defaults.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ALPHA_MIN = 1e-4  # material.py:21

EXTENSION_DEFAULTS = {
    "coat_weight": 0.0,
    "coat_roughness": 0.0,
    "coat_ior": 1.5,
    "coat_color": (1.0, 1.0, 1.0),
    "transmission_weight": 0.0,
    "transmission_color": (1.0, 1.0, 1.0),
}


def _in_unit(name: str, v: float) -> None:
    if not 0.0 <= v <= 1.0:
        raise ValueError(f"{name} must lie in [0, 1], got {v!r}")


@dataclass(frozen=True)
class OpenPbrParams:
    base_weight: float = 1.0
    base_color: tuple[float, float, float] = (0.8, 0.8, 0.8)
    base_metalness: float = 0.0
    specular_weight: float = 1.0
    specular_color: tuple[float, float, float] = (1.0, 1.0, 1.0)
    specular_roughness: float = 0.3
    specular_ior: float = 1.5
    emission_luminance: float = 0.0
    emission_color: tuple[float, float, float] = (1.0, 1.0, 1.0)
    # extensions (no reference implementation; parity unpinned)
    coat_weight: float = 0.0
    coat_roughness: float = 0.0
    coat_ior: float = 1.5
    coat_color: tuple[float, float, float] = (1.0, 1.0, 1.0)
    transmission_weight: float = 0.0
    transmission_color: tuple[float, float, float] = (1.0, 1.0, 1.0)

    def __post_init__(self) -> None:
        for name in ("base_weight", "base_metalness", "specular_weight", "specular_roughness",
                     "coat_weight", "coat_roughness", "transmission_weight"):
            _in_unit(name, getattr(self, name))
        for name in ("base_color", "specular_color", "emission_color", "coat_color",
                     "transmission_color"):
            c = getattr(self, name)
            if len(c) != 3 or any(not 0.0 <= x <= 1.0 for x in c):
                raise ValueError(f"{name} must be three channels in [0, 1], got {c!r}")
        if self.specular_ior < 1.0:
            raise ValueError(f"specular_ior must be >= 1, got {self.specular_ior!r}")
        if self.coat_ior < 1.0:
            raise ValueError(f"coat_ior must be >= 1, got {self.coat_ior!r}")
        if self.emission_luminance < 0.0:
            raise ValueError(f"emission_luminance must be >= 0, got {self.emission_luminance!r}")


def emitted_radiance(params) -> np.ndarray:
    return params.emission_luminance * np.asarray(params.emission_color, dtype=np.float64)


def pack_materials(materials):
    """The reference's 9-array SoA packing (material.py:68-92), same order
    (fresh, writable arrays, as the reference returns)."""
    mats = list(materials)
    if not mats:
        raise ValueError("scene has no materials")
    t = _pack_material_table(mats)
    return (t["base_weight"], t["base_color"], t["base_metalness"], t["specular_weight"],
            t["specular_color"], t["specular_roughness"], t["specular_ior"],
            t["emission_luminance"], t["emission_color"])


_SCALARS = ("base_weight", "base_metalness", "specular_weight", "specular_roughness",
            "specular_ior", "emission_luminance", "coat_weight", "coat_roughness", "coat_ior",
            "transmission_weight")
_COLORS = ("base_color", "specular_color", "emission_color", "coat_color", "transmission_color")


_TABLES: dict = {}


def pack_material_table(materials) -> dict[str, np.ndarray]:
    """All material arrays (reference + extension) keyed by field name;
    (k,) or (k, 3) float64, C-contiguous.  Memoized for hashable (frozen)
    material objects; the arrays are shared, read-only."""
    mats = list(materials)
    if not mats:
        raise ValueError("scene has no materials")
    try:
        key = tuple(mats)
        hit = _TABLES.get(key)
    except TypeError:           # unhashable material objects: no memo
        return _pack_material_table(mats)
    if hit is None:
        if len(_TABLES) >= 64:
            _TABLES.clear()
        hit = _TABLES[key] = _pack_material_table(mats)
        for a in hit.values():
            a.flags.writeable = False
    return hit


def _pack_material_table(mats) -> dict[str, np.ndarray]:
    out = {}
    for name in _SCALARS:
        out[name] = np.array([float(getattr(m, name, EXTENSION_DEFAULTS.get(name, 0.0)))
                              for m in mats], dtype=np.float64)
    for name in _COLORS:
        out[name] = np.ascontiguousarray(
            [tuple(getattr(m, name, EXTENSION_DEFAULTS.get(name))) for m in mats],
            dtype=np.float64).reshape(len(mats), 3)
    return out


def has_extensions(materials) -> bool:
    return any(float(getattr(m, "coat_weight", 0.0)) > 0.0
               or float(getattr(m, "transmission_weight", 0.0)) > 0.0 for m in materials)
