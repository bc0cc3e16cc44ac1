"""Synthetic workloads of the benchmark and the tests (BASELINE.json configs
C1-C5).

  * cornell_box      C1/C2: ~36 axis-aligned triangles on a dyadic grid (all
                     coordinates exact in fp32), diffuse walls, emissive quad;
                     variant "mixed" adds metal / glossy-dielectric boxes,
                     variant "extended" adds coat / glass (extensions).
  * sphere_on_plane  C3: `bumpy_sphere(70_000)` on a 2-triangle metal plane
                     under the reference's benchmark gradient sky.
  * pushbutton       C4/C5: a CAD-style pushbutton assembly of ~1.06 M
                     triangles (housing, knurled collar, chrome bezel,
                     coated cap, glass lens, LED ring, base plate, screws)
                     with mixed OpenPBR materials.
  * synthetic_hdr    equirectangular sky + sun radiance map (extension).

Pure numpy: this module never imports the product package, so the CPU
reference arm (`bench.py --impl reference`) builds exactly the same scenes
without loading the product library.  The objects duck-type the
reference's render inputs (luxtrace SceneDescription / TriangleBuffer /
OpenPbrParams / CameraConfig / EnvironmentConfig, scene.py:52-111,510-516,
geometry.py:88-131, material.py:25-53), which both the product's
DeviceScene and the oracle accept.

Vertices are rounded to float32 (as a GLB stores them, procgen.py:123 of the
reference) so the float64 oracle and the fp32 kernels see identical
positions.  Everything is deterministic.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BENCH_ENVIRONMENT = dict(zenith=(0.5, 0.6, 0.9), horizon=(0.9, 0.85, 0.8))  # bench.py:33-34


# ------------------------------------------------------------------ render inputs

@dataclass
class Triangles:
    """TriangleBuffer layout (geometry.py:88-131): (n, 3) float64 arrays."""
    v0: np.ndarray
    v1: np.ndarray
    v2: np.ndarray
    n0: np.ndarray
    n1: np.ndarray
    n2: np.ndarray
    material_index: np.ndarray

    def __len__(self) -> int:
        return int(self.v0.shape[0])


@dataclass(frozen=True)
class Material:
    """OpenPbrParams fields (material.py:25-53) + the coat / transmission
    extensions (zero weight = the reference material)."""
    base_weight: float = 1.0
    base_color: tuple = (0.8, 0.8, 0.8)
    base_metalness: float = 0.0
    specular_weight: float = 1.0
    specular_color: tuple = (1.0, 1.0, 1.0)
    specular_roughness: float = 0.3
    specular_ior: float = 1.5
    emission_luminance: float = 0.0
    emission_color: tuple = (1.0, 1.0, 1.0)
    coat_weight: float = 0.0
    coat_roughness: float = 0.0
    coat_ior: float = 1.5
    coat_color: tuple = (1.0, 1.0, 1.0)
    transmission_weight: float = 0.0
    transmission_color: tuple = (1.0, 1.0, 1.0)


@dataclass
class Camera:
    """CameraConfig fields (scene.py:52-81)."""
    position: tuple
    look_at: tuple
    up: tuple = (0.0, 1.0, 0.0)
    vertical_fov_deg: float = 45.0
    width: int = 512
    height: int = 512


@dataclass
class Environment:
    """EnvironmentConfig fields (scene.py:84-111) + the lat-long extension."""
    kind: str
    radiance: np.ndarray = field(default_factory=lambda: np.zeros(3))
    zenith: np.ndarray = field(default_factory=lambda: np.zeros(3))
    horizon: np.ndarray = field(default_factory=lambda: np.zeros(3))
    texels: np.ndarray | None = None
    scale: float = 1.0

    @classmethod
    def uniform(cls, radiance) -> "Environment":
        return cls("uniform", radiance=np.asarray(radiance, np.float64))

    @classmethod
    def gradient(cls, zenith, horizon) -> "Environment":
        return cls("gradient", zenith=np.asarray(zenith, np.float64),
                   horizon=np.asarray(horizon, np.float64))

    @classmethod
    def latlong(cls, texels, scale: float = 1.0) -> "Environment":
        return cls("latlong", texels=np.ascontiguousarray(texels, np.float32), scale=float(scale))


@dataclass
class Scene:
    """SceneDescription fields (scene.py:510-516)."""
    triangles: Triangles
    materials: list
    camera: Camera
    environment: Environment
    degenerate_dropped: int = 0
    parts: list | None = None     # MeshBuilder parts (indexed meshes), for write_gltf


# ------------------------------------------------------------------ meshes

def smooth_normals(positions: np.ndarray, indices: np.ndarray) -> np.ndarray:
    """Area-weighted vertex normals (scene.py:493-507 semantics)."""
    a, b, c = (positions[indices[k::3]] for k in range(3))
    face = np.cross(b - a, c - a)
    acc = np.zeros_like(positions)
    for k in range(3):
        np.add.at(acc, indices[k::3], face)
    length = np.linalg.norm(acc, axis=1, keepdims=True)
    zero = length[:, 0] == 0.0
    acc[zero] = (0.0, 0.0, 1.0)
    length[zero] = 1.0
    return acc / length


def bumpy_sphere(n_triangles: int, bump_amplitude: float = 0.12,
                 bump_frequencies=(6.0, 4.0), radius: float = 1.0):
    """Displaced lat/long sphere with exactly n_triangles faces: the reference
    generator's surface (procgen.py:71-114), as paper_2407_19977_b200.procgen
    has it (kept here so this module needs no product import)."""
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


class MeshBuilder:
    """Collects indexed parts, emits a Triangles buffer with per-corner
    normals (smooth within a part, float32-rounded positions)."""

    def __init__(self):
        self.parts = []

    def add(self, positions, indices, material: int, normals=None):
        positions = np.asarray(positions, dtype=np.float32).astype(np.float64)
        indices = np.asarray(indices, dtype=np.int64).ravel()
        if normals is None:
            normals = smooth_normals(positions, indices)
        self.parts.append((positions, indices, np.asarray(normals, np.float64), int(material)))
        return self

    def add_flat(self, tris, material: int):
        """tris: (k, 3, 3) corner positions; flat (face) normals."""
        tris = np.asarray(tris, dtype=np.float32).astype(np.float64)
        fn = np.cross(tris[:, 1] - tris[:, 0], tris[:, 2] - tris[:, 0])
        fn /= np.linalg.norm(fn, axis=1, keepdims=True)
        pos = tris.reshape(-1, 3)
        idx = np.arange(pos.shape[0])
        return self.add(pos, idx, material, normals=np.repeat(fn, 3, axis=0))

    def build(self) -> Triangles:
        cols = {k: [] for k in ("v0", "v1", "v2", "n0", "n1", "n2")}
        mats = []
        for pos, idx, nrm, mat in self.parts:
            for k in range(3):
                cols[f"v{k}"].append(pos[idx[k::3]])
                cols[f"n{k}"].append(nrm[idx[k::3]])
            mats.append(np.full(idx.size // 3, mat, np.int32))
        return Triangles(*(np.vstack(cols[k]) for k in ("v0", "v1", "v2", "n0", "n1", "n2")),
                         material_index=np.concatenate(mats))

    @property
    def n_triangles(self) -> int:
        return sum(p[1].size // 3 for p in self.parts)


def quad(a, b, c, d):
    """Two triangles (a, b, c), (a, c, d)."""
    return [[a, b, c], [a, c, d]]


def box_tris(lo, hi):
    x0, y0, z0 = lo
    x1, y1, z1 = hi
    p = [(x0, y0, z0), (x1, y0, z0), (x1, y1, z0), (x0, y1, z0),
         (x0, y0, z1), (x1, y0, z1), (x1, y1, z1), (x0, y1, z1)]
    faces = [(0, 3, 2, 1), (4, 5, 6, 7), (0, 1, 5, 4), (3, 7, 6, 2), (0, 4, 7, 3), (1, 2, 6, 5)]
    out = []
    for a, b, c, d in faces:   # outward winding
        out += quad(p[a], p[b], p[c], p[d])
    return out


def revolve(profile_r, profile_y, n_theta: int, radial=None):
    """Surface of revolution about +y: profile (r_j, y_j), j = 0..m-1,
    n_theta segments; `radial(theta, j)` optionally multiplies r.  Returns
    (positions, indices) with a duplicated seam (outward winding for a
    profile that runs bottom -> top on the outside)."""
    r = np.asarray(profile_r, np.float64)
    y = np.asarray(profile_y, np.float64)
    m = r.size
    th = np.linspace(0.0, 2.0 * math.pi, n_theta + 1)
    R = np.broadcast_to(r[None, :], (n_theta + 1, m)).copy()
    if radial is not None:
        R = R * radial(th[:, None], np.arange(m)[None, :])
    pos = np.stack([R * np.cos(th)[:, None], np.broadcast_to(y[None, :], R.shape),
                    -R * np.sin(th)[:, None]], axis=-1).reshape(-1, 3)
    i = np.arange(n_theta)[:, None] * m
    j = np.arange(m - 1)[None, :]
    a = i + j
    b = a + m
    lo = np.stack([a, b, a + 1], -1).reshape(-1, 3)
    hi = np.stack([a + 1, b, b + 1], -1).reshape(-1, 3)
    faces = np.empty((2 * lo.shape[0], 3), np.int64)
    faces[0::2], faces[1::2] = lo, hi
    return pos, faces.ravel()


def torus(R: float, r: float, y0: float, n_theta: int, n_phi: int):
    ph = np.linspace(0.0, 2.0 * math.pi, n_phi + 1)
    return revolve(R + r * np.cos(ph), y0 + r * np.sin(ph), n_theta)


# ------------------------------------------------------------------ scenes

def cornell_box(width: int = 64, height: int = 64, variant: str = "diffuse") -> Scene:
    """Cornell-style box on a dyadic grid.  variant: 'diffuse' (C1),
    'mixed' (metal + glossy dielectric boxes, reference lobes only), or
    'extended' (coat + glass boxes: extension lobes)."""
    white = Material(base_color=(0.75, 0.75, 0.75), specular_weight=0.0)
    red = Material(base_color=(0.75, 0.125, 0.125), specular_weight=0.0)
    green = Material(base_color=(0.125, 0.75, 0.125), specular_weight=0.0)
    light = Material(base_color=(0.75, 0.75, 0.75), specular_weight=0.0,
                          emission_luminance=15.0, emission_color=(1.0, 0.875, 0.75))
    if variant == "diffuse":
        tall = short = white
    elif variant == "mixed":
        tall = Material(base_color=(0.875, 0.75, 0.5), base_metalness=1.0,
                             specular_roughness=0.125)
        short = Material(base_color=(0.25, 0.375, 0.75), specular_roughness=0.25,
                              specular_ior=1.5)
    elif variant == "extended":
        tall = Material(base_color=(0.875, 0.75, 0.5), base_metalness=1.0,
                             specular_roughness=0.125)
        short = Material(base_color=(0.75, 0.125, 0.0625), specular_roughness=0.375,
                              coat_weight=1.0, coat_roughness=0.0625)
        glass = Material(base_color=(1.0, 1.0, 1.0), specular_roughness=0.0625,
                              transmission_weight=1.0, transmission_color=(0.875, 0.9375, 1.0))
    else:
        raise ValueError(f"unknown cornell variant {variant!r}")
    mats = [white, red, green, light, tall, short]
    mb = MeshBuilder()
    s = 1.0
    h = 2.0
    walls = []
    walls += quad((-s, 0, -s), (s, 0, -s), (s, 0, s), (-s, 0, s))      # floor (y=0, faces +y)
    walls += quad((-s, h, -s), (-s, h, s), (s, h, s), (s, h, -s))      # ceiling
    walls += quad((-s, 0, -s), (-s, h, -s), (s, h, -s), (s, 0, -s))    # back
    mb.add_flat(walls, 0)
    mb.add_flat(quad((-s, 0, -s), (-s, 0, s), (-s, h, s), (-s, h, -s)), 1)   # left (red)
    mb.add_flat(quad((s, 0, -s), (s, h, -s), (s, h, s), (s, 0, s)), 2)       # right (green)
    ly = 1.984375
    mb.add_flat(quad((-0.25, ly, -0.25), (0.25, ly, -0.25), (0.25, ly, 0.25), (-0.25, ly, 0.25)),
                3)
    mb.add_flat(box_tris((-0.625, 0.0, -0.625), (-0.125, 1.25, -0.125)), 4)   # tall box
    mb.add_flat(box_tris((0.125, 0.0, -0.125), (0.625, 0.625, 0.375)), 5)     # short box
    if variant == "extended":
        mats.append(glass)
        mb.add_flat(box_tris((-0.5, 0.0, 0.25), (-0.125, 0.375, 0.625)), 6)   # glass block
    cam = Camera(position=(0.0, 1.0, 3.75), look_at=(0.0, 1.0, 0.0),
                       vertical_fov_deg=40.0, width=width, height=height)
    return Scene(mb.build(), mats, cam, Environment.uniform((0.0, 0.0, 0.0)), parts=mb.parts)


def sphere_on_plane(n_triangles: int = 70_000, width: int = 1920, height: int = 1080,
                    environment=None) -> Scene:
    """C3: bumpy_sphere(n) resting above a 2-triangle metal ground plane."""
    pos, idx = bumpy_sphere(n_triangles)
    pos = pos + np.array([0.0, 1.125, 0.0])
    mb = MeshBuilder()
    mb.add(pos, idx, 0)
    g = 16.0
    mb.add_flat(quad((-g, 0, -g), (-g, 0, g), (g, 0, g), (g, 0, -g)), 1)
    mats = [Material(base_color=(0.8, 0.55, 0.45), specular_roughness=0.4),
            Material(base_color=(0.9, 0.9, 0.92), base_metalness=1.0,
                          specular_roughness=0.2)]
    cam = Camera(position=(0.0, 1.5, 4.75), look_at=(0.0, 1.0, 0.0),
                       vertical_fov_deg=40.0, width=width, height=height)
    env = environment or Environment.gradient(**BENCH_ENVIRONMENT)
    return Scene(mb.build(), mats, cam, env, parts=mb.parts)


def pushbutton(width: int = 1920, height: int = 1080, extended: bool = True,
               environment=None, detail: float = 0.807) -> Scene:
    """C4: CAD-style pushbutton assembly, ~1.07 M triangles at the default detail.
    extended=False swaps the coat / glass materials for reference lobes (the
    parity-pinned variant)."""
    def n(x):
        return max(8, int(round(x * detail)))

    mats = [
        Material(base_color=(0.35, 0.36, 0.38), specular_roughness=0.55),          # 0 ground
        Material(base_color=(0.91, 0.92, 0.92), base_metalness=1.0,
                      specular_roughness=0.35),                                          # 1 housing
        Material(base_color=(0.56, 0.57, 0.58), base_metalness=1.0,
                      specular_roughness=0.25),                                          # 2 knurl
        Material(base_color=(0.97, 0.96, 0.91), base_metalness=1.0,
                      specular_roughness=0.06),                                          # 3 bezel
        Material(base_color=(0.8, 0.05, 0.04), specular_roughness=0.35,
                      coat_weight=1.0 if extended else 0.0, coat_roughness=0.05),        # 4 cap
        Material(base_color=(0.95, 0.97, 1.0), specular_roughness=0.02,
                      specular_weight=1.0,
                      transmission_weight=1.0 if extended else 0.0,
                      transmission_color=(0.9, 0.95, 1.0)),                              # 5 lens
        Material(base_color=(0.2, 0.9, 0.3), specular_weight=0.0,
                      emission_luminance=8.0, emission_color=(0.2, 1.0, 0.35)),          # 6 LED
        Material(base_color=(0.04, 0.04, 0.045), specular_roughness=0.5),           # 7 plate
        Material(base_color=(0.75, 0.75, 0.77), base_metalness=1.0,
                      specular_roughness=0.2),                                           # 8 screws
    ]
    mb = MeshBuilder()
    # ground
    g = 24.0
    mb.add_flat(quad((-g, 0, -g), (-g, 0, g), (g, 0, g), (g, 0, -g)), 0)
    # base plate and four screws
    mb.add_flat(box_tris((-1.6, 0.0, -1.6), (1.6, 0.12, 1.6)), 7)
    for sx, sz in ((-1.3, -1.3), (1.3, -1.3), (-1.3, 1.3), (1.3, 1.3)):
        ph = np.linspace(0.0, 0.5 * math.pi, n(24))
        prof_r = np.concatenate([[0.0], 0.11 * np.cos(ph[::-1])])
        prof_y = np.concatenate([[0.12], 0.12 + 0.05 * np.sin(ph[::-1])])
        pos, idx = revolve(prof_r[::-1], prof_y[::-1], n(192))
        mb.add(pos + np.array([sx, 0.0, sz]), idx, 8)
    # housing: cylinder with a rounded top edge, y in [0.12, 0.75]
    t = np.linspace(0.0, 1.0, n(96))
    edge = np.linspace(0.0, 0.5 * math.pi, n(48))
    hr = np.concatenate([np.full(t.size, 1.0), 0.92 + 0.08 * np.cos(edge[1:]),
                         np.linspace(0.92, 0.86, n(8))[1:]])
    hy = np.concatenate([0.12 + 0.55 * t, 0.67 + 0.08 * np.sin(edge[1:]),
                         np.full(n(8) - 1, 0.75)])
    pos, idx = revolve(hr, hy, n(1536))
    mb.add(pos, idx, 1)
    # knurled collar: radius modulated by 60 ridges
    kt = np.linspace(0.0, 1.0, n(40))
    ridges = 60

    def knurl(theta, j):
        return 1.0 + 0.018 * np.abs(np.cos(0.5 * ridges * theta))

    pos, idx = revolve(np.full(kt.size, 1.02), 0.2 + 0.3 * kt, n(3072), radial=knurl)
    mb.add(pos, idx, 2)
    # chrome bezel: torus
    pos, idx = torus(0.86, 0.07, 0.76, n(1536), n(96))
    mb.add(pos, idx, 3)
    # LED ring
    pos, idx = torus(0.74, 0.018, 0.77, n(1024), n(24))
    mb.add(pos, idx, 6)
    # cap: rippled dome over r in [0, 0.7]
    ct = np.linspace(0.0, 1.0, n(160))
    cr = 0.7 * np.sin(0.5 * math.pi * (1.0 - ct))
    cy = 0.78 + 0.22 * np.sin(0.5 * math.pi * ct)

    def ripple(theta, j):
        return 1.0 + 0.01 * np.sin(12.0 * theta) * np.sin(math.pi * np.clip(j / (ct.size - 1), 0, 1))

    pos, idx = revolve(cr[::-1], cy[::-1], n(1536), radial=ripple)
    mb.add(pos, idx, 4)
    # glass lens over the cap top
    lt = np.linspace(0.0, 1.0, n(48))
    lr = 0.3 * np.cos(0.5 * math.pi * lt)
    ly = 1.015 + 0.06 * np.sin(0.5 * math.pi * lt)
    pos, idx = revolve(lr, ly, n(768))
    mb.add(pos, idx, 5)
    cam = Camera(position=(0.0, 2.6, 3.9), look_at=(0.0, 0.55, 0.0),
                       vertical_fov_deg=34.0, width=width, height=height)
    env = environment
    if env is None:
        env = Environment.latlong(synthetic_hdr(), 1.0) if extended else \
            Environment.gradient(**BENCH_ENVIRONMENT)
    return Scene(mb.build(), mats, cam, env, parts=mb.parts)


def synthetic_hdr(width: int = 1024, height: int = 512, sun_dir=(0.45, 0.6, 0.35),
                  sun_radiance: float = 400.0, sun_angle_deg: float = 2.5) -> np.ndarray:
    """Equirectangular (height, width, 3) float32 radiance: a vertical sky
    gradient, a warm horizon band, a dark ground and a small bright sun --
    the dynamic range of a captured HDR sky (extension; no reference)."""
    v = (np.arange(height) + 0.5) / height
    u = (np.arange(width) + 0.5) / width
    theta = v * math.pi                       # 0 at zenith
    phi = (u - 0.5) * 2.0 * math.pi
    st, ct = np.sin(theta)[:, None], np.cos(theta)[:, None]
    d = np.stack([st * np.sin(phi)[None, :], np.broadcast_to(ct, (height, width)),
                  -st * np.cos(phi)[None, :]], axis=-1)
    y = d[..., 1:2]
    zen = np.array([0.25, 0.45, 1.0])
    hor = np.array([1.0, 0.85, 0.65])
    ground = np.array([0.18, 0.16, 0.14])
    sky = hor + (zen - hor) * np.clip(y, 0.0, 1.0) ** 0.5
    img = np.where(y >= 0.0, sky, ground * (1.0 + 0.5 * np.clip(-y, 0.0, 1.0)))
    s = np.asarray(sun_dir, np.float64)
    s /= np.linalg.norm(s)
    cosang = np.tensordot(d, s, axes=([2], [0]))
    core = np.cos(math.radians(sun_angle_deg))
    halo = np.clip((cosang - 0.9) / 0.1, 0.0, 1.0) ** 8
    img = img + (cosang >= core)[..., None] * sun_radiance * np.array([1.0, 0.95, 0.85])
    img = img + halo[..., None] * np.array([2.0, 1.8, 1.4])
    return np.ascontiguousarray(img, dtype=np.float32)


def write_gltf(scene: Scene, glb_path, config_path, normals: bool = True) -> None:
    """The scene as a GLB + render config that `load_scene` reads: one mesh
    per MeshBuilder part (float32 positions, float32 normals unless
    `normals` is False -- then the loader generates smooth normals -- and
    u32 indices), material "m<k>" bound in the config to the scene's k-th
    material, one identity node per mesh.  A lat-long environment is written
    as uniform white (the config format has no maps)."""
    import json
    import struct
    from dataclasses import asdict
    blobs, views, accessors, meshes, nodes, used = [], [], [], [], [], {}
    offset = 0

    def add_blob(arr, ctype, kind, count):
        nonlocal offset
        data = arr.tobytes()
        views.append({"buffer": 0, "byteOffset": offset, "byteLength": len(data)})
        blobs.append(data + b"\x00" * (-len(data) % 4))
        offset += len(blobs[-1])
        accessors.append({"bufferView": len(views) - 1, "componentType": ctype,
                          "count": int(count), "type": kind})
        return len(accessors) - 1

    for pos, idx, nrm, mat in scene.parts:
        attrs = {"POSITION": add_blob(np.asarray(pos, np.float32), 5126, "VEC3", len(pos))}
        if normals:
            attrs["NORMAL"] = add_blob(np.asarray(nrm, np.float32), 5126, "VEC3", len(pos))
        ind = add_blob(np.asarray(idx, np.uint32), 5125, "SCALAR", idx.size)
        used.setdefault(mat, len(used))
        meshes.append({"primitives": [{"attributes": attrs, "indices": ind,
                                       "material": used[mat]}]})
        nodes.append({"mesh": len(meshes) - 1})
    binary = b"".join(blobs)
    doc = {"asset": {"version": "2.0"}, "buffers": [{"byteLength": len(binary)}],
           "bufferViews": views, "accessors": accessors, "meshes": meshes, "nodes": nodes,
           "scenes": [{"nodes": list(range(len(nodes)))}], "scene": 0,
           "materials": [{"name": f"m{m}"} for m in used]}
    js = json.dumps(doc).encode()
    js += b" " * (-len(js) % 4)
    with open(glb_path, "wb") as f:
        f.write(struct.pack("<III", 0x46546C67, 2, 28 + len(js) + len(binary)))
        f.write(struct.pack("<II", len(js), 0x4E4F534A) + js)
        f.write(struct.pack("<II", len(binary), 0x004E4942) + binary)
    cam, env = scene.camera, scene.environment
    if env.kind == "gradient":
        env_doc = {"type": "gradient", "zenith": [float(x) for x in env.zenith],
                   "horizon": [float(x) for x in env.horizon]}
    elif env.kind == "uniform":
        env_doc = {"type": "uniform", "radiance": [float(x) for x in env.radiance]}
    else:
        env_doc = {"type": "uniform", "radiance": [1.0, 1.0, 1.0]}
    config = {"camera": {"position": [float(x) for x in cam.position],
                         "look_at": [float(x) for x in cam.look_at],
                         "up": [float(x) for x in cam.up],
                         "vertical_fov_deg": float(cam.vertical_fov_deg),
                         "width": int(cam.width), "height": int(cam.height)},
              "environment": env_doc,
              "materials": {f"m{m}": {k: (list(v) if isinstance(v, tuple) else v)
                                      for k, v in asdict(scene.materials[m]).items()}
                            for m in used}}
    with open(config_path, "w") as f:
        json.dump(config, f)


def scene_by_name(name: str, **kw) -> Scene:
    """Named workloads used by bench.py and the tests."""
    if name == "cornell_c1":
        return cornell_box(kw.get("width", 64), kw.get("height", 64), "diffuse")
    if name == "cornell_c2":
        return cornell_box(kw.get("width", 512), kw.get("height", 512), "mixed")
    if name == "cornell_c2x":
        return cornell_box(kw.get("width", 512), kw.get("height", 512), "extended")
    if name == "sphere70k":
        return sphere_on_plane(kw.get("n_triangles", 70_000), kw.get("width", 1920),
                               kw.get("height", 1080))
    if name == "pushbutton":
        return pushbutton(kw.get("width", 1920), kw.get("height", 1080), True,
                          detail=kw.get("detail", 0.807))
    if name == "pushbutton_ref":
        return pushbutton(kw.get("width", 1920), kw.get("height", 1080), False,
                          detail=kw.get("detail", 0.807))
    raise ValueError(f"unknown scene {name!r}")
