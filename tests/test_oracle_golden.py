"""Pin the CPU oracle (oracle/lt_oracle.c) to the reference's own outputs.

The golden fixtures were produced by running the reference (make_golden.py).
The oracle restates the reference term for term in float64, so every check
here is exact equality (bit-for-bit), not a tolerance.
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import GOLDEN, golden_scene

KAT = [2707161783, 2068313097, 3122475824, 2211639955, 3215226955, 3421331566, 3217466285,
       2167406445]   # test_rng.py:14-24


def test_pcg_known_answer(oracle_lib):
    st, inc = oracle_lib.pcg_seed(42, 54)
    out = []
    for _ in range(8):
        v, st = oracle_lib.pcg_next(st, inc)
        out.append(v)
    assert out == KAT
    z = np.load(GOLDEN / "rng.npz")
    assert out == z["kat_42_54"].tolist()


def test_seed_stream_matches_reference(oracle_lib):
    z = np.load(GOLDEN / "rng.npz")
    for (pix, smp, seed), (gs, gi), draws in zip(z["stream_keys"].tolist(),
                                                 z["stream_states"].tolist(),
                                                 z["stream_draws"].tolist()):
        st, inc = oracle_lib.seed_stream(pix, smp, seed)
        assert (st, inc) == (gs, gi)
        got = []
        for _ in range(6):
            v, st = oracle_lib.pcg_next(st, inc)
            got.append(v)
        assert got == draws


def test_material_sampling_matches_reference(oracle_lib):
    z = np.load(GOLDEN / "material.npz")
    names = ("base_weight", "c0", "c1", "c2", "base_metalness", "specular_weight", "s0", "s1",
             "s2", "specular_roughness", "specular_ior")
    mismatches = 0
    for prm, row in zip(z["params"], z["rows"]):
        class P:  # noqa: N801 - attribute bag
            pass
        p = P()
        d = dict(zip(names, prm))
        p.base_weight, p.base_metalness = d["base_weight"], d["base_metalness"]
        p.base_color = (d["c0"], d["c1"], d["c2"])
        p.specular_weight, p.specular_roughness = d["specular_weight"], d["specular_roughness"]
        p.specular_color = (d["s0"], d["s1"], d["s2"])
        p.specular_ior = d["specular_ior"]
        wo, n, u = row[0:3], row[3:6], row[6:9]
        ok_ref = row[9] > 0.5
        ok, wi, w, pdf, spike = oracle_lib.sample_bsdf(wo, n, p, u)
        assert ok == ok_ref
        if ok:
            if not (np.array_equal(wi, row[10:13]) and np.array_equal(w, row[13:16])
                    and pdf == row[16] and spike == (row[17] > 0.5)):
                mismatches += 1
        f = oracle_lib.eval_bsdf(wo, row[18:21], n, p)
        assert np.array_equal(f, row[21:24])
        assert oracle_lib.pdf_bsdf(wo, row[18:21], n, p) == row[24]
    assert mismatches == 0


@pytest.mark.parametrize("name", ["floor", "shell", "glossy", "sphere2k", "dup", "cornell_c1",
                                  "cornell_c2", "sphere20k"])
def test_oracle_traversal_bit_exact(name, oracle_lib):
    g = golden_scene(name)
    oc = g.oracle()
    idx, t = oc.intersect_batch(g["rays_o"], g["rays_d"])
    assert np.array_equal(idx, g["isect_idx"])
    assert np.array_equal(t, g["isect_t"])
    bi, bt = oc.brute_force_batch(g["rays_o"], g["rays_d"])
    assert np.array_equal(bi, g["brute_idx"])
    assert np.array_equal(bt, g["brute_t"])
    nodes, tests = oc.traversal_counts(g["rays_o"], g["rays_d"])
    assert np.array_equal(nodes, g["count_nodes"])
    assert np.array_equal(tests, g["count_tests"])


@pytest.mark.parametrize("name", ["floor", "shell", "glossy", "sphere2k", "dup", "cornell_c1",
                                  "cornell_c2", "sphere20k"])
def test_oracle_render_bit_exact(name, oracle_lib):
    """_render_pass restated: full render and per-sample values identical."""
    g = golden_scene(name)
    oc = g.oracle()
    w, h = g.camera.width, g.camera.height
    s = g.settings
    acc = np.zeros((h, w, 3))
    val = np.zeros((h, w), np.int64)
    inv = np.zeros((h, w), np.int64)
    oc.render_pass(acc, val, inv, 0, s.samples_per_pixel, g["cam_pack"], w, h, s.seed,
                   s.max_depth, s.rr_start_depth, s.t_min)
    assert np.array_equal(acc, g["render_image"])
    assert np.array_equal(inv, g["render_invalid"])
    pix = np.arange(w * h)
    for k, ref in enumerate(g["per_sample"]):
        rgb, seg = oc.sample_values(pix, k, g["cam_pack"], w, h, s.seed, s.max_depth,
                                    s.rr_start_depth, s.t_min)
        ref = ref.reshape(-1, 3)
        finite = np.isfinite(ref).all(axis=1)
        assert np.array_equal(rgb[finite], ref[finite])
        assert np.all(seg >= 1) and np.all(seg <= s.max_depth)


@pytest.mark.parametrize("name", ["floor", "glossy", "sphere2k", "cornell_c2"])
def test_oracle_trace_radiance_bit_exact(name, oracle_lib):
    g = golden_scene(name)
    oc = g.oracle()
    s = g.settings
    for k, ((st, inc), rgb_ref, st_ref) in enumerate(zip(g["trace_state_in"].tolist(),
                                                         g["trace_rgb"],
                                                         g["trace_state_out"].tolist())):
        rgb, st_out, _ = oc.trace(g["rays_o"][k], g["rays_d"][k], st, inc, s.max_depth,
                                  s.rr_start_depth, s.t_min)
        assert np.array_equal(rgb, rgb_ref)
        assert st_out == st_ref


def test_oracle_chunking_invariant(oracle_lib):
    g = golden_scene("glossy")
    oc = g.oracle()
    w, h = g.camera.width, g.camera.height
    s = g.settings
    a = [np.zeros((h, w, 3)), np.zeros((h, w), np.int64), np.zeros((h, w), np.int64)]
    b = [np.zeros((h, w, 3)), np.zeros((h, w), np.int64), np.zeros((h, w), np.int64)]
    oc.render_pass(*a, 0, 6, g["cam_pack"], w, h, s.seed, s.max_depth, s.rr_start_depth)
    for start in range(0, 6, 2):
        oc.render_pass(*b, start, 2, g["cam_pack"], w, h, s.seed, s.max_depth, s.rr_start_depth,
                       threads=3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("name", ["floor", "shell", "glossy", "sphere2k", "dup", "cornell_c1",
                                  "cornell_c2", "sphere20k"])
def test_oracle_bvh_build_bit_exact(name, oracle_lib):
    """oc_build_bvh (the reference arm's tree) == luxtrace.build_bvh's arrays."""
    g = golden_scene(name)
    b = oracle_lib.build_bvh(g.triangles)
    assert np.array_equal(b.bounds_min, g["bvh_bounds_min"])
    assert np.array_equal(b.bounds_max, g["bvh_bounds_max"])
    for mine, ref in (("left_child", "bvh_left"), ("right_child", "bvh_right"),
                      ("first_triangle", "bvh_first"), ("triangle_count", "bvh_count"),
                      ("triangle_order", "bvh_order")):
        assert np.array_equal(getattr(b, mine), g[ref]), mine


@pytest.mark.parametrize("name", ["floor", "glossy", "cornell_c2"])
def test_oracle_camera_pack_matches_reference(name, oracle_lib):
    g = golden_scene(name)
    assert np.array_equal(oracle_lib.camera_pack(g.camera), g["cam_pack"])
