"""ctypes wrapper of the CPU fp64 oracle (oracle/lt_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py (cpu_baseline leg and --impl reference).  Never by the product
package.  The oracle restates the reference (file:line cited in the C
source) and is pinned against golden vectors produced by the reference
itself (tests/golden/make_golden.py).
"""
from __future__ import annotations

import ctypes as C
import math
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "_build" / "liblt_oracle.so"

_dp = C.POINTER(C.c_double)
_fp = C.POINTER(C.c_float)
_ip = C.POINTER(C.c_int32)
_lp = C.POINTER(C.c_int64)
_up = C.POINTER(C.c_uint64)


class OcScene(C.Structure):
    _fields_ = [
        ("n_nodes", C.c_int64), ("bmin", _dp), ("bmax", _dp),
        ("left", _ip), ("right", _ip), ("first", _ip), ("count", _ip), ("order", _ip),
        ("n_tris", C.c_int64),
        ("v0", _dp), ("v1", _dp), ("v2", _dp), ("n0", _dp), ("n1", _dp), ("n2", _dp),
        ("mat_index", _ip),
        ("n_mats", C.c_int32),
        ("bw", _dp), ("bc", _dp), ("metal", _dp), ("sw", _dp), ("sc", _dp), ("rough", _dp),
        ("ior", _dp), ("el", _dp), ("ec", _dp),
        ("coat_w", _dp), ("coat_rough", _dp), ("coat_ior", _dp), ("coat_color", _dp),
        ("tr_w", _dp), ("tr_color", _dp),
        ("env_kind", C.c_int32),
        ("env_a", C.c_double * 3), ("env_b", C.c_double * 3),
        ("env_w", C.c_int32), ("env_h", C.c_int32),
        ("env_map", _fp),
        ("env_scale", C.c_double),
    ]


_lib = None


def build() -> Path:
    """Compile the oracle (make -C oracle); a no-op when up to date."""
    subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            build()
        h = C.CDLL(str(LIB_PATH))
        h.oc_pcg_next.restype = C.c_uint32
        h.oc_pcg_next.argtypes = [_up, C.c_uint64]
        h.oc_pcg_seed.argtypes = [C.c_uint64, C.c_uint64, _up, _up]
        h.oc_mix64.restype = C.c_uint64
        h.oc_mix64.argtypes = [C.c_uint64]
        h.oc_seed_stream.argtypes = [C.c_uint64, C.c_uint64, C.c_uint64, _up, _up]
        sp = C.POINTER(OcScene)
        h.oc_intersect_batch.argtypes = [sp, _dp, _dp, C.c_int64, C.c_double, C.c_double, _lp,
                                         _dp, C.c_int]
        h.oc_traversal_counts_batch.argtypes = [sp, _dp, _dp, C.c_int64, C.c_double, C.c_double,
                                                _lp, _lp, C.c_int]
        h.oc_brute_force_batch.argtypes = [sp, _dp, _dp, C.c_int64, C.c_double, C.c_double, _lp,
                                           _dp, C.c_int]
        h.oc_eval_bsdf.argtypes = [_dp, _dp, _dp, _dp, _dp]
        h.oc_pdf_bsdf.restype = C.c_double
        h.oc_pdf_bsdf.argtypes = [_dp, _dp, _dp, _dp]
        h.oc_sample_bsdf.restype = C.c_int
        h.oc_sample_bsdf.argtypes = [_dp, _dp, _dp, C.c_double, C.c_double, C.c_double, C.c_int,
                                     _dp, _dp, _dp, C.POINTER(C.c_int)]
        h.oc_camera_dir.argtypes = [_dp, C.c_double, C.c_double, C.c_double, C.c_double,
                                    C.c_int32, C.c_int32, _dp]
        h.oc_trace.restype = C.c_int
        h.oc_trace.argtypes = [sp, _dp, _dp, _up, C.c_uint64, C.c_int32, C.c_int32, C.c_double,
                               _dp]
        h.oc_render_pass.argtypes = [sp, _dp, _lp, _lp, C.c_int64, C.c_int64, _dp, C.c_int32,
                                     C.c_int32, C.c_uint64, C.c_int32, C.c_int32, C.c_double,
                                     C.c_int, _lp]
        h.oc_sample_values.argtypes = [sp, _lp, C.c_int64, C.c_int64, _dp, C.c_int32, C.c_int32,
                                       C.c_uint64, C.c_int32, C.c_int32, C.c_double, _dp, _ip,
                                       C.c_int]
        h.oc_primary_rays.argtypes = [_lp, C.c_int64, C.c_int64, _dp, C.c_int32, C.c_int32,
                                      C.c_uint64, _dp, _dp]
        h.oc_mt_intersect.restype = C.c_int
        h.oc_mt_intersect.argtypes = [_dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double, _dp, _dp,
                                      _dp]
        h.oc_slab_intersect.restype = C.c_int
        h.oc_slab_intersect.argtypes = [_dp, _dp, _dp, _dp, C.c_double, C.c_double, _dp, _dp]
        h.oc_hit_frame_api.argtypes = [_dp, _dp, _dp, _dp, _dp, _dp, _dp, C.c_double, C.c_double,
                                       _dp, _dp, C.POINTER(C.c_int)]
        h.oc_build_bvh.restype = C.c_int64
        h.oc_build_bvh.argtypes = [_dp, _dp, _dp, C.c_int64, C.c_int32, C.c_int32, _dp, _dp,
                                   _ip, _ip, _ip, _ip, _ip, _lp, _lp]
        _lib = h
    return _lib


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


def default_threads() -> int:
    return int(os.environ.get("ORACLE_THREADS", os.cpu_count() or 1))


# ------------------------------------------------------------------ rng

def pcg_seed(init_state: int, init_seq: int) -> tuple[int, int]:
    s, i = C.c_uint64(), C.c_uint64()
    lib().oc_pcg_seed(init_state & (2**64 - 1), init_seq & (2**64 - 1), C.byref(s), C.byref(i))
    return s.value, i.value


def pcg_next(state: int, inc: int) -> tuple[int, int]:
    s = C.c_uint64(state)
    out = lib().oc_pcg_next(C.byref(s), inc)
    return int(out), s.value


def seed_stream(pixel: int, sample: int, seed: int) -> tuple[int, int]:
    s, i = C.c_uint64(), C.c_uint64()
    lib().oc_seed_stream(pixel, sample, seed & (2**64 - 1), C.byref(s), C.byref(i))
    return s.value, i.value


# ------------------------------------------------------------------ geometry

def _v(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def mt_intersect(o, d, a, b, c, t_min, t_max):
    """_mt_intersect (geometry.py:138-167): (hit, t, u, v)."""
    t, u, v = C.c_double(), C.c_double(), C.c_double()
    ok = lib().oc_mt_intersect(*[_p(_v(x), C.c_double) for x in (o, d, a, b, c)], float(t_min),
                               float(t_max), C.byref(t), C.byref(u), C.byref(v))
    return bool(ok), t.value, u.value, v.value


def slab_intersect(o, d, lo, hi, t_min, t_max):
    """ray_aabb_intersect's arithmetic (geometry.py:244-248, 170-207):
    (hit, t_enter, t_exit)."""
    inv = np.array([np.inf if x == 0.0 else 1.0 / x for x in np.asarray(d, np.float64)])
    tn, tf = C.c_double(), C.c_double()
    ok = lib().oc_slab_intersect(_p(_v(o), C.c_double), _p(inv, C.c_double),
                                 _p(_v(lo), C.c_double), _p(_v(hi), C.c_double), float(t_min),
                                 float(t_max), C.byref(tn), C.byref(tf))
    return bool(ok), tn.value, tf.value


def hit_frame(d, a, b, c, n0, n1, n2, u, v):
    """_hit_frame (geometry.py:210-241): (geometric, shading, front)."""
    g, s = np.zeros(3), np.zeros(3)
    fr = C.c_int()
    lib().oc_hit_frame_api(*[_p(_v(x), C.c_double) for x in (d, a, b, c, n0, n1, n2)], float(u),
                           float(v), _p(g, C.c_double), _p(s, C.c_double), C.byref(fr))
    return g, s, bool(fr.value)


# ------------------------------------------------------------------ camera

def camera_pack(camera) -> np.ndarray:
    """_camera_pack (integrator.py:75-83): [position, forward, right, up,
    tan(fov/2), aspect], the reference's numpy operations in order."""
    def unit(v):
        return v / np.linalg.norm(v)
    position = np.asarray(camera.position, dtype=np.float64)
    forward = unit(np.asarray(camera.look_at, dtype=np.float64) - position)
    right = unit(np.cross(forward, np.asarray(camera.up, dtype=np.float64)))
    up = np.cross(right, forward)
    tan_half = math.tan(math.radians(camera.vertical_fov_deg) * 0.5)
    return np.ascontiguousarray(np.concatenate([position, forward, right, up,
                                                [tan_half, camera.width / camera.height]]))


# ------------------------------------------------------------------ bvh build

class OracleBvh:
    """The reference's Bvh arrays (bvh.py:38-50) from oc_build_bvh, the C
    restatement of build_bvh (bvh.py:286-298)."""

    def __init__(self, bounds_min, bounds_max, left_child, right_child, first_triangle,
                 triangle_count, triangle_order, leaf_count, max_depth):
        self.bounds_min, self.bounds_max = bounds_min, bounds_max
        self.left_child, self.right_child = left_child, right_child
        self.first_triangle, self.triangle_count = first_triangle, triangle_count
        self.triangle_order = triangle_order
        self.leaf_count, self.max_depth = leaf_count, max_depth


def build_bvh(triangles, leaf_size: int = 4, bins: int = 12) -> OracleBvh:
    v0, v1, v2 = (np.ascontiguousarray(getattr(triangles, k), dtype=np.float64).reshape(-1, 3)
                  for k in ("v0", "v1", "v2"))
    n = v0.shape[0]
    if n == 0:
        raise ValueError("empty scene")
    m = 2 * n
    bmin, bmax = np.empty((m, 3)), np.empty((m, 3))
    ints = [np.empty(m, np.int32) for _ in range(4)]
    order = np.empty(n, np.int32)
    leaves, depth = C.c_int64(), C.c_int64()
    nn = lib().oc_build_bvh(_p(v0, C.c_double), _p(v1, C.c_double), _p(v2, C.c_double), n,
                            int(leaf_size), int(bins), _p(bmin, C.c_double),
                            _p(bmax, C.c_double), *[_p(a, C.c_int32) for a in ints],
                            _p(order, C.c_int32), C.byref(leaves), C.byref(depth))
    if nn < 0:
        raise MemoryError("oc_build_bvh: allocation failed")
    return OracleBvh(bmin[:nn].copy(), bmax[:nn].copy(), *[a[:nn].copy() for a in ints], order,
                     int(leaves.value), int(depth.value))


# ------------------------------------------------------------------ materials

def material_params(p) -> np.ndarray:
    """21-vector of oc_* material params from an OpenPbrParams-like object."""
    g = lambda n, d: getattr(p, n, d)
    return np.array([g("base_weight", 1.0), *g("base_color", (0.8,) * 3), g("base_metalness", 0.0),
                     g("specular_weight", 1.0), *g("specular_color", (1.0,) * 3),
                     g("specular_roughness", 0.3), g("specular_ior", 1.5),
                     g("coat_weight", 0.0), g("coat_roughness", 0.0), g("coat_ior", 1.5),
                     *g("coat_color", (1.0,) * 3), g("transmission_weight", 0.0),
                     *g("transmission_color", (1.0,) * 3)], dtype=np.float64)


def eval_bsdf(wo, wi, n, params) -> np.ndarray:
    f = np.zeros(3)
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (wo, wi, n)]
    pr = material_params(params)
    lib().oc_eval_bsdf(*(_p(x, C.c_double) for x in a), _p(pr, C.c_double), _p(f, C.c_double))
    return f


def pdf_bsdf(wo, wi, n, params) -> float:
    a = [np.ascontiguousarray(x, dtype=np.float64) for x in (wo, wi, n)]
    pr = material_params(params)
    return float(lib().oc_pdf_bsdf(*(_p(x, C.c_double) for x in a), _p(pr, C.c_double)))


def sample_bsdf(wo, n, params, draws, front: bool = True):
    """(ok, wi, weight, pdf, spike)"""
    wo = np.ascontiguousarray(wo, dtype=np.float64)
    n = np.ascontiguousarray(n, dtype=np.float64)
    pr = material_params(params)
    wi, w, pdf = np.zeros(3), np.zeros(3), np.zeros(1)
    spike = C.c_int()
    ok = lib().oc_sample_bsdf(_p(wo, C.c_double), _p(n, C.c_double), _p(pr, C.c_double),
                              float(draws[0]), float(draws[1]), float(draws[2]), int(front),
                              _p(wi, C.c_double), _p(w, C.c_double), _p(pdf, C.c_double),
                              C.byref(spike))
    return bool(ok), wi, w, float(pdf[0]), bool(spike.value)


# ------------------------------------------------------------------ scenes

_EXT_FIELDS = {"coat_weight": 0.0, "coat_roughness": 0.0, "coat_ior": 1.5,
               "transmission_weight": 0.0}


class OracleScene:
    """oc_scene over numpy arrays (kept alive by this object)."""

    def __init__(self, triangles, bvh, materials, environment):
        self._keep = []
        s = OcScene()

        def d(a, shape=None):
            arr = np.ascontiguousarray(a, dtype=np.float64)
            if shape is not None:
                arr = arr.reshape(shape)
            self._keep.append(arr)
            return _p(arr, C.c_double)

        def i(a):
            arr = np.ascontiguousarray(a, dtype=np.int32)
            self._keep.append(arr)
            return _p(arr, C.c_int32)

        nn = len(bvh.left_child)
        s.n_nodes = nn
        s.bmin, s.bmax = d(bvh.bounds_min, (nn, 3)), d(bvh.bounds_max, (nn, 3))
        s.left, s.right = i(bvh.left_child), i(bvh.right_child)
        s.first, s.count, s.order = i(bvh.first_triangle), i(bvh.triangle_count), \
            i(bvh.triangle_order)
        t = triangles
        s.n_tris = len(t.v0)
        s.v0, s.v1, s.v2, s.n0, s.n1, s.n2 = (d(getattr(t, k)) for k in
                                              ("v0", "v1", "v2", "n0", "n1", "n2"))
        s.mat_index = i(t.material_index)
        mats = list(materials)
        s.n_mats = len(mats)
        g = lambda name, dflt: [getattr(m, name, dflt) for m in mats]
        s.bw = d(g("base_weight", 1.0))
        s.bc = d(g("base_color", (0.8,) * 3), (len(mats), 3))
        s.metal = d(g("base_metalness", 0.0))
        s.sw = d(g("specular_weight", 1.0))
        s.sc = d(g("specular_color", (1.0,) * 3), (len(mats), 3))
        s.rough = d(g("specular_roughness", 0.3))
        s.ior = d(g("specular_ior", 1.5))
        s.el = d(g("emission_luminance", 0.0))
        s.ec = d(g("emission_color", (1.0,) * 3), (len(mats), 3))
        s.coat_w = d(g("coat_weight", 0.0))
        s.coat_rough = d(g("coat_roughness", 0.0))
        s.coat_ior = d(g("coat_ior", 1.5))
        s.coat_color = d(g("coat_color", (1.0,) * 3), (len(mats), 3))
        s.tr_w = d(g("transmission_weight", 0.0))
        s.tr_color = d(g("transmission_color", (1.0,) * 3), (len(mats), 3))
        env = environment
        if env.kind == "uniform":
            s.env_kind = 0
            s.env_a[:] = list(map(float, env.radiance))
            s.env_b[:] = list(map(float, env.radiance))
        elif env.kind == "gradient":
            s.env_kind = 1
            s.env_a[:] = list(map(float, env.zenith))
            s.env_b[:] = list(map(float, env.horizon))
        else:
            s.env_kind = 2
            tex = np.ascontiguousarray(env.texels, dtype=np.float32)
            self._keep.append(tex)
            s.env_h, s.env_w = tex.shape[0], tex.shape[1]
            s.env_map = _p(tex, C.c_float)
            s.env_scale = float(env.scale)
        self.struct = s
        self.ref = C.byref(s)

    @classmethod
    def from_scene(cls, scene, bvh):
        return cls(scene.triangles, bvh, scene.materials, scene.environment)

    # -- queries
    def intersect_batch(self, origins, dirs, t_min=1e-4, t_max=np.inf, threads=None):
        o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        dd = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
        idx = np.empty(o.shape[0], np.int64)
        t = np.empty(o.shape[0])
        lib().oc_intersect_batch(self.ref, _p(o, C.c_double), _p(dd, C.c_double), o.shape[0],
                                 t_min, t_max, _p(idx, C.c_int64), _p(t, C.c_double),
                                 threads or default_threads())
        return idx, t

    def brute_force_batch(self, origins, dirs, t_min=1e-4, t_max=np.inf, threads=None):
        o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        dd = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
        idx = np.empty(o.shape[0], np.int64)
        t = np.empty(o.shape[0])
        lib().oc_brute_force_batch(self.ref, _p(o, C.c_double), _p(dd, C.c_double), o.shape[0],
                                   t_min, t_max, _p(idx, C.c_int64), _p(t, C.c_double),
                                   threads or default_threads())
        return idx, t

    def traversal_counts(self, origins, dirs, t_min=1e-4, t_max=np.inf, threads=None):
        o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
        dd = np.ascontiguousarray(dirs, dtype=np.float64).reshape(-1, 3)
        nodes = np.empty(o.shape[0], np.int64)
        tests = np.empty(o.shape[0], np.int64)
        lib().oc_traversal_counts_batch(self.ref, _p(o, C.c_double), _p(dd, C.c_double),
                                        o.shape[0], t_min, t_max, _p(nodes, C.c_int64),
                                        _p(tests, C.c_int64), threads or default_threads())
        return nodes, tests

    def trace(self, origin, direction, state, inc, max_depth, rr_start, t_min=1e-4):
        o = np.ascontiguousarray(origin, dtype=np.float64)
        dd = np.ascontiguousarray(direction, dtype=np.float64)
        st = C.c_uint64(state)
        rgb = np.zeros(3)
        seg = lib().oc_trace(self.ref, _p(o, C.c_double), _p(dd, C.c_double), C.byref(st), inc,
                             max_depth, rr_start, t_min, _p(rgb, C.c_double))
        return rgb, st.value, int(seg)

    def render_pass(self, accum, valid, invalid, sample_start, sample_count, cam, width, height,
                    seed, max_depth, rr_start, t_min=1e-4, threads=None):
        """In-place `_render_pass`; returns the closest-hit queries issued."""
        cam = np.ascontiguousarray(cam, dtype=np.float64)
        seg = C.c_int64()
        lib().oc_render_pass(self.ref, _p(accum, C.c_double), _p(valid, C.c_int64),
                             _p(invalid, C.c_int64), sample_start, sample_count,
                             _p(cam, C.c_double), width, height, seed, max_depth, rr_start, t_min,
                             threads or default_threads(), C.byref(seg))
        return int(seg.value)

    def sample_values(self, pixels, sample, cam, width, height, seed, max_depth, rr_start,
                      t_min=1e-4, threads=None):
        pix = np.ascontiguousarray(pixels, dtype=np.int64)
        cam = np.ascontiguousarray(cam, dtype=np.float64)
        rgb = np.zeros((pix.size, 3))
        seg = np.zeros(pix.size, np.int32)
        lib().oc_sample_values(self.ref, _p(pix, C.c_int64), pix.size, sample,
                               _p(cam, C.c_double), width, height, seed, max_depth, rr_start,
                               t_min, _p(rgb, C.c_double), _p(seg, C.c_int32),
                               threads or default_threads())
        return rgb, seg


def primary_rays(pixels, sample, cam, width, height, seed):
    pix = np.ascontiguousarray(pixels, dtype=np.int64)
    cam = np.ascontiguousarray(cam, dtype=np.float64)
    o = np.zeros((pix.size, 3))
    d = np.zeros((pix.size, 3))
    lib().oc_primary_rays(_p(pix, C.c_int64), pix.size, sample, _p(cam, C.c_double), width,
                          height, seed, _p(o, C.c_double), _p(d, C.c_double))
    return o, d
