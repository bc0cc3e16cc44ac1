"""The GPU BVH build (csrc/lt_bvh_gpu.cu, row (f)2 of SURVEY §8) against the
reference's build_bvh (bvh.py:286-298).

* CPU: the closed form of the reference's in-place two-pointer partition
  (bvh.py:224-238) that the GPU evaluates with prefix sums, checked against
  the sequential procedure on every flag pattern up to 12 elements.
* GPU: `build_bvh(device=0)` returns exactly the reference's arrays on every
  golden scene (reference-built fixtures) and the same arrays as the host
  restatement on larger and degenerate scenes (coincident centroids -> the
  median split, flat scenes -> zero-area leaves, odd leaf sizes / bin
  counts).
"""
from __future__ import annotations

import itertools
import zlib

import numpy as np
import pytest

from conftest import SCENES, golden_scene


def two_pointer(a, right):
    """bvh.py:224-238 restated: i from the left, j from the right, swap."""
    a = list(a)
    i, j = 0, len(a) - 1
    while i <= j:
        if not right[a[i]]:
            i += 1
        else:
            a[i], a[j] = a[j], a[i]
            j -= 1
    return a, i


def closed_form(a, right):
    """The GPU's permutation (lt_bvh_gpu.cu scatter_one) from prefix counts."""
    c = len(a)
    flag = [0 if right[x] else 1 for x in a]           # 1 = left
    pre = np.concatenate([[0], np.cumsum(flag)]).astype(int)
    L = int(pre[c])
    beta, belem = [0] * c, [0] * c
    for k in range(L, c):
        if flag[k]:
            jj = 1 + (pre[c] - pre[k + 1])
            beta[jj - 1] = c - k
            belem[jj - 1] = a[k]
    X = L - int(pre[L])
    last = beta[X - 1] if X > 0 else 0
    out = [None] * c
    for k in range(c):
        x = a[k]
        if k < L:
            if flag[k]:
                out[k] = x
            else:
                jj = 1 + (k - int(pre[k]))
                out[k] = belem[jj - 1]
                out[c - 1 - (beta[jj - 2] if jj >= 2 else 0)] = x
        elif not flag[k]:
            p = c - k
            out[(k - 1) if p < last else (c - 1 - last if k == L else k - 1)] = x
    return out, L


def test_partition_closed_form_is_exhaustively_exact():
    for c in range(1, 13):
        a = list(range(c))
        for bits in itertools.product([False, True], repeat=c):
            right = dict(zip(a, bits))
            assert closed_form(a, right) == two_pointer(a, right), (c, bits)


def _same(a, b):
    assert a.stats.node_count == b.stats.node_count
    assert a.stats.leaf_count == b.stats.leaf_count
    assert a.stats.max_depth == b.stats.max_depth
    for name in ["bounds_min", "bounds_max", "left_child", "right_child", "first_triangle",
                 "triangle_count", "triangle_order"]:
        x, y = getattr(a, name), getattr(b, name)
        assert x.shape == y.shape, name
        assert np.array_equal(x, y), name   # == on floats: +-0 compare equal


@pytest.mark.gpu
@pytest.mark.parametrize("name", SCENES)
def test_gpu_build_equals_reference(name):
    from paper_2407_19977_b200 import build_bvh
    g = golden_scene(name)
    b = build_bvh(g.triangles, device=0)
    assert np.array_equal(b.bounds_min, g["bvh_bounds_min"])
    assert np.array_equal(b.bounds_max, g["bvh_bounds_max"])
    assert np.array_equal(b.left_child, g["bvh_left"])
    assert np.array_equal(b.right_child, g["bvh_right"])
    assert np.array_equal(b.first_triangle, g["bvh_first"])
    assert np.array_equal(b.triangle_count, g["bvh_count"])
    assert np.array_equal(b.triangle_order, g["bvh_order"])


def _soup(n, rng, coincident=0, flat=False):
    """Random triangles; `coincident` copies of one triangle (identical
    centroids force the median split); `flat` puts everything in z = 0."""
    from paper_2407_19977_b200 import TriangleBuffer
    c = rng.uniform(-10, 10, (n, 3))
    v0 = c + rng.normal(0, 0.3, (n, 3))
    v1 = c + rng.normal(0, 0.3, (n, 3))
    v2 = c + rng.normal(0, 0.3, (n, 3))
    if coincident:
        v0[:coincident], v1[:coincident], v2[:coincident] = v0[0], v1[0], v2[0]
    if flat:
        for v in (v0, v1, v2):
            v[:, 2] = 0.0
    nrm = np.tile([0.0, 0.0, 1.0], (n, 1))
    return TriangleBuffer(v0, v1, v2, nrm, nrm, nrm, np.zeros(n, np.int32))


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["tiny1", "tiny5", "soup3k", "soup20k", "soup200k",
                                  "coincident", "flat", "leaf1", "leaf7", "bins2", "bins32"])
def test_gpu_build_equals_host_build(case):
    from paper_2407_19977_b200 import build_bvh
    rng = np.random.default_rng(zlib.crc32(case.encode()))
    kw = {}
    if case == "tiny1":
        tris = _soup(1, rng)
    elif case == "tiny5":
        tris = _soup(5, rng)
    elif case == "soup3k":
        tris = _soup(3000, rng)
    elif case == "soup20k":
        tris = _soup(20000, rng)
    elif case == "soup200k":
        tris = _soup(200000, rng)
    elif case == "coincident":
        tris = _soup(30000, rng, coincident=9000)
    elif case == "flat":
        tris = _soup(20000, rng, flat=True)
    elif case == "leaf1":
        tris, kw = _soup(10000, rng), {"leaf_size": 1}
    elif case == "leaf7":
        tris, kw = _soup(10000, rng), {"leaf_size": 7}
    elif case == "bins2":
        tris, kw = _soup(10000, rng), {"bins": 2}
    else:
        tris, kw = _soup(50000, rng), {"bins": 32}
    _same(build_bvh(tris, device=0, **kw), build_bvh(tris, device=None, **kw))


@pytest.mark.gpu
@pytest.mark.parametrize("scene", ["pushbutton", "sphere70k"])
def test_gpu_build_equals_host_build_bench_scenes(scene):
    """The bench workloads (1.06 M and 70 k triangles)."""
    import time
    from paper_2407_19977_b200 import build_bvh
    from workloads import scene_by_name
    tris = scene_by_name(scene, width=64, height=36).triangles
    build_bvh(tris, device=0)   # warm (module load, allocations)
    t0 = time.perf_counter()
    gpu = build_bvh(tris, device=0)
    t_gpu = time.perf_counter() - t0
    t0 = time.perf_counter()
    host = build_bvh(tris, device=None)
    t_host = time.perf_counter() - t0
    print(f"{scene}: {len(tris)} triangles, GPU build {1e3 * t_gpu:.1f} ms, "
          f"host build {1e3 * t_host:.1f} ms")
    _same(gpu, host)
