"""Render inputs of the drop-in API: camera, environment, scene description.

Mirrors luxtrace.scene's render-input types (scene.py:52-111, 510-516) and
_camera_pack / _environment_pack (integrator.py:75-83, 118-121).  glTF
ingest stays out of scope: a SceneDescription built by the
reference's loader is accepted unchanged.

Extension: EnvironmentConfig.latlong(texels, scale) -- an equirectangular
HDR map (the north star's synthetic HDR environment; parity unpinned).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .geometry import TriangleBuffer, normalize


class SceneError(ValueError):
    """Malformed or unsupported scene input (scene.py:44-45)."""


@dataclass
class CameraConfig:
    position: np.ndarray
    look_at: np.ndarray
    up: np.ndarray = field(default_factory=lambda: np.array([0.0, 1.0, 0.0]))
    vertical_fov_deg: float = 45.0
    width: int = 512
    height: int = 512

    def __post_init__(self) -> None:
        for name in ("position", "look_at", "up"):
            v = np.asarray(getattr(self, name), dtype=np.float64)
            if v.shape != (3,) or not np.all(np.isfinite(v)):
                raise SceneError(f"camera {name} must be three finite numbers, got {v!r}")
            setattr(self, name, v)
        forward = self.look_at - self.position
        if float(np.linalg.norm(forward)) == 0.0:
            raise SceneError("camera position and look_at must differ")
        if float(np.linalg.norm(self.up)) == 0.0:
            raise SceneError("camera up must be non-zero")
        if float(np.linalg.norm(np.cross(forward, self.up))) < 1e-9:
            raise SceneError("camera up must not be parallel to the view direction")
        if not 0.0 < self.vertical_fov_deg < 180.0:
            raise SceneError(f"vertical_fov_deg must lie in (0, 180), got {self.vertical_fov_deg}")
        self.width, self.height = int(self.width), int(self.height)
        if self.width < 1 or self.height < 1:
            raise SceneError("image width and height must be >= 1")


@dataclass
class EnvironmentConfig:
    """'uniform' radiance, a 'gradient' horizon -> zenith over d.y in [0, 1],
    or (extension) a 'latlong' equirectangular radiance map."""

    kind: str
    radiance: np.ndarray = field(default_factory=lambda: np.zeros(3))
    zenith: np.ndarray = field(default_factory=lambda: np.zeros(3))
    horizon: np.ndarray = field(default_factory=lambda: np.zeros(3))
    texels: np.ndarray | None = None      # (h, w, 3) float32, latlong only
    scale: float = 1.0

    def __post_init__(self) -> None:
        if self.kind not in ("uniform", "gradient", "latlong"):
            raise SceneError(f"environment type must be 'uniform' or 'gradient' (or the "
                             f"'latlong' extension), got {self.kind!r}")
        for name in ("radiance", "zenith", "horizon"):
            v = np.asarray(getattr(self, name), dtype=np.float64)
            if v.shape != (3,) or np.any(v < 0.0) or not np.all(np.isfinite(v)):
                raise SceneError(f"environment {name} must be three non-negative numbers")
            setattr(self, name, v)
        if self.kind == "latlong":
            t = np.ascontiguousarray(self.texels, dtype=np.float32)
            if t.ndim != 3 or t.shape[2] != 3 or t.shape[0] < 1 or t.shape[1] < 1:
                raise SceneError("latlong texels must have shape (h, w, 3)")
            if np.any(t < 0.0) or not np.all(np.isfinite(t)):
                raise SceneError("latlong texels must be finite and non-negative")
            self.texels = t
            if not (self.scale >= 0.0 and math.isfinite(self.scale)):
                raise SceneError("latlong scale must be finite and non-negative")

    @classmethod
    def uniform(cls, radiance) -> "EnvironmentConfig":
        return cls(kind="uniform", radiance=np.asarray(radiance, dtype=np.float64))

    @classmethod
    def gradient(cls, zenith, horizon) -> "EnvironmentConfig":
        return cls(kind="gradient", zenith=np.asarray(zenith, dtype=np.float64),
                   horizon=np.asarray(horizon, dtype=np.float64))

    @classmethod
    def latlong(cls, texels, scale: float = 1.0) -> "EnvironmentConfig":
        return cls(kind="latlong", texels=texels, scale=float(scale))


@dataclass
class SceneDescription:
    triangles: TriangleBuffer
    materials: list
    camera: CameraConfig
    environment: EnvironmentConfig
    degenerate_dropped: int = 0


_CAMERA_PACKS: dict = {}


def camera_pack(camera) -> np.ndarray:
    """[position, forward, right, up, tan(fov/2), aspect] -- the 14 doubles of
    _camera_pack (integrator.py:75-83), same numpy operations.  Memoized by
    the camera's values (a dozen small numpy calls cost ~0.1 ms, a visible
    share of a small render call); a copy is returned."""
    try:
        key = (tuple(float(x) for x in camera.position),
               tuple(float(x) for x in camera.look_at), tuple(float(x) for x in camera.up),
               float(camera.vertical_fov_deg), int(camera.width), int(camera.height))
    except (TypeError, ValueError):
        return _camera_pack(camera)
    hit = _CAMERA_PACKS.get(key)
    if hit is None:
        if len(_CAMERA_PACKS) >= 64:
            _CAMERA_PACKS.clear()
        hit = _CAMERA_PACKS[key] = _camera_pack(camera)
    return hit.copy()


def _camera_pack(camera) -> np.ndarray:
    position = np.asarray(camera.position, dtype=np.float64)
    forward = normalize(np.asarray(camera.look_at, dtype=np.float64) - position)
    right = normalize(np.cross(forward, np.asarray(camera.up, dtype=np.float64)))
    cam_up = np.cross(right, forward)
    tan_half = math.tan(math.radians(camera.vertical_fov_deg) * 0.5)
    aspect = camera.width / camera.height
    return np.ascontiguousarray(np.concatenate([position, forward, right, cam_up,
                                                [tan_half, aspect]]), dtype=np.float64)


ENV_KINDS = {"uniform": 0, "gradient": 1, "latlong": 2}


def environment_pack(env):
    """(kind, a, b) as _environment_pack (integrator.py:118-121)."""
    kind = env.kind
    if kind == "uniform":
        r = np.asarray(env.radiance, dtype=np.float64)
        return 0, r.copy(), r.copy()
    if kind == "gradient":
        return 1, np.asarray(env.zenith, dtype=np.float64).copy(), \
            np.asarray(env.horizon, dtype=np.float64).copy()
    if kind == "latlong":
        return 2, np.zeros(3), np.zeros(3)
    raise SceneError(f"unknown environment kind {kind!r}")
