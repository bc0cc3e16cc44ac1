"""Parity on the headline configuration (BASELINE.json configs[3], C4): the
1.06 M-triangle pushbutton at 1920x1080, depth 8, against the float64 oracle
at matched RNG streams -- every pixel of the full frame, two samples each.

  * `pushbutton_ref` (reference lobes, gradient sky): the pinned parity case.
    Per (pixel, sample): |gpu - oracle| <= 1e-4 * max(1, |oracle|) for
    >= 99.9 % of rows; rows whose primary ray hits a
    near-mirror lobe (alpha = max(roughness^2, 1e-4) < 0.01: the chrome
    bezel, the lens) are counted separately -- a 1-ulp change of the hit
    point moves a D ~ 1/alpha^2 spike sample across the lobe;
  * `pushbutton` (the bench scene: coat, glass, HDR sky; parity unpinned,
    the oracle's own float64 implementation of the same estimator);
  * primary-hit triangle ids over the full frame, mismatches counted.

Every measurement is appended to gpurun_out/parity_r02.jsonl
(tools/parity_report.py -> profiles/parity_r02.json).
"""
from __future__ import annotations

import numpy as np
import pytest

from conftest import agreement_tiers, record_parity

pytestmark = pytest.mark.gpu

W, H = 1920, 1080
_scenes: dict = {}


def headline(name: str):
    """(scene, bvh, DeviceScene, OracleScene, packed camera), cached."""
    if name not in _scenes:
        import paper_2407_19977_b200 as m
        from oracle.oracle import OracleScene
        from workloads import scene_by_name
        sc = scene_by_name(name, width=W, height=H)
        bvh = m.build_bvh(sc.triangles)
        _scenes[name] = (sc, bvh, m.DeviceScene(sc, bvh), OracleScene.from_scene(sc, bvh),
                         m.camera_pack(sc.camera))
    return _scenes[name]


def gpu_sample(ds, camera, settings, sample):
    from paper_2407_19977_b200.integrator import Accumulator, render_pass_device
    acc = Accumulator(camera.width, camera.height, ds.device)
    render_pass_device(ds, camera, settings, acc, sample, 1)
    v = acc.valid.cpu().numpy()
    s = acc.sum.view(-1, 3).double().cpu().numpy()
    s[v == 0] = np.nan
    return s


def primary_alpha(sc, oc, cam, sample, seed):
    """alpha of the material the primary ray of every pixel hits (inf on a
    miss)."""
    from oracle.oracle import primary_rays
    o, d = primary_rays(np.arange(W * H), sample, cam, W, H, seed)
    idx, _ = oc.intersect_batch(o, d)
    rough = np.array([float(m.specular_roughness) for m in sc.materials])
    metal = np.array([float(m.base_metalness) for m in sc.materials])
    spec = np.array([float(m.specular_weight) for m in sc.materials])
    alpha = np.maximum(rough ** 2, 1e-4)
    # a diffuse-only material (no metal, no specular) has no glossy lobe
    alpha = np.where((metal <= 0) & (spec <= 0), np.inf, alpha)
    mi = np.asarray(sc.triangles.material_index)
    out = np.full(W * H, np.inf)
    hit = idx >= 0
    out[hit] = alpha[mi[idx[hit]]]
    return out


@pytest.mark.parametrize("name", ["pushbutton_ref", "pushbutton"])
def test_headline_per_sample_parity(name):
    import paper_2407_19977_b200 as m
    sc, bvh, ds, oc, cam = headline(name)
    st = m.RenderSettings(samples_per_pixel=1, max_depth=8, rr_start_depth=3, seed=0)
    gots, refs, mirror = [], [], []
    for s in range(2):
        ref, _ = oc.sample_values(np.arange(W * H), s, cam, W, H, st.seed, st.max_depth,
                                  st.rr_start_depth, st.t_min)
        gots.append(gpu_sample(ds, sc.camera, st, s))
        refs.append(ref)
        mirror.append(primary_alpha(sc, oc, cam, s, st.seed) < 0.01)
    got, ref, mirror = np.concatenate(gots), np.concatenate(refs), np.concatenate(mirror)
    all_rows = agreement_tiers(got, ref)
    rest = agreement_tiers(got[~mirror], ref[~mirror])
    near_mirror = agreement_tiers(got[mirror], ref[mirror])
    record_parity("headline_per_sample", scene=name, triangles=len(sc.triangles),
                  width=W, height=H, samples=2, max_depth=8, all=all_rows,
                  excluding_near_mirror=rest, near_mirror_primary=near_mirror,
                  near_mirror_rows=int(mirror.sum()))
    print(name, "all", all_rows, "\nnear-mirror", near_mirror)
    assert rest["frac_le_0.0001"] >= 0.999
    assert all_rows["frac_le_0.001"] >= 0.995
    assert all_rows["nonfinite_mismatch"] == 0


def edge_margin(tris, k, o, d):
    """float64 plane hit of ray (o, d) with triangle k: (t, signed distance
    of the hit point to the triangle's boundary in world units, >= 0 inside;
    |cos| of the ray against the plane)."""
    a, b, c = tris.v0[k], tris.v1[k], tris.v2[k]
    n = np.cross(b - a, c - a)
    n /= np.linalg.norm(n)
    cos = abs(float(np.dot(d, n)))
    t = np.dot(a - o, n) / np.dot(d, n)
    p = o + t * d
    margin = np.inf
    for u, v, w in ((a, b, c), (b, c, a), (c, a, b)):
        e = np.cross(n, v - u)
        e /= np.linalg.norm(e)
        if np.dot(w - u, e) < 0:
            e = -e
        margin = min(margin, float(np.dot(p - u, e)))
    return float(t), margin, cos


def classify_mismatch(tris, o, d, ours, ref):
    """A mismatch is ulp-level when, in float64, the two candidates are a
    near-tie in t or one of them is hit within EPS of its boundary (an
    edge or vertex shared by neighbours).  EPS = 1e-6 (|o| + t) / |cos|:
    ~10 float32 ulps of the coordinates, times the conditioning of the
    ray-plane intersection (a grazing ray moves its plane hit point by
    1/|cos| per unit of error along the ray)."""
    t_o, m_o, c_o = edge_margin(tris, ours, o, d)
    t_r, m_r, c_r = edge_margin(tris, ref, o, d)
    scale = 1e-6 * (np.abs(o).max() + max(abs(t_o), abs(t_r)))
    eps_o, eps_r = scale / max(c_o, 1e-3), scale / max(c_r, 1e-3)
    edge = abs(m_o) <= eps_o or abs(m_r) <= eps_r
    return {"tie": abs(t_o - t_r) <= scale, "edge": edge, "dt": abs(t_o - t_r),
            "margin": min(abs(m_o), abs(m_r)), "eps": min(eps_o, eps_r),
            "cos": (c_o, c_r)}


def test_headline_primary_hit_ids():
    """Full-frame primary-hit ids on the 1.06 M-triangle scene vs the
    float64 oracle traversal of the same jittered rays; every mismatch is
    classified in float64 as an edge or tie case."""
    import paper_2407_19977_b200 as m
    from oracle.oracle import primary_rays
    sc, bvh, ds, oc, cam = headline("pushbutton_ref")
    total, mism_total, unexplained = 0, 0, []
    for s in range(2):
        o, d = primary_rays(np.arange(W * H), s, cam, W, H, 0)
        ref_i, ref_t = oc.intersect_batch(o, d)
        idx, t = m.intersect_scene_batch(sc.triangles, bvh, o, d, scene=ds)
        bad = np.nonzero(idx != ref_i)[0]
        flips = int(np.sum((idx >= 0) != (ref_i >= 0)))
        kinds = [classify_mismatch(sc.triangles, o[r], d[r], idx[r], ref_i[r])
                 for r in bad if idx[r] >= 0 and ref_i[r] >= 0]
        edge = sum(k["edge"] for k in kinds)
        tie = sum(k["tie"] and not k["edge"] for k in kinds)
        unexplained += [k for k in kinds if not (k["edge"] or k["tie"])]
        same = (idx == ref_i) & (ref_i >= 0)
        rel_t = float(np.max(np.abs(t[same] - ref_t[same]) / np.maximum(1.0, ref_t[same])))
        total += idx.size
        mism_total += bad.size
        record_parity("headline_primary_ids", scene="pushbutton_ref", sample=s, rays=idx.size,
                      id_mismatches=int(bad.size), ppm=1e6 * bad.size / idx.size,
                      max_rel_t=rel_t, hit_miss_flips=flips, edge_cases=int(edge),
                      tie_cases=int(tie),
                      max_margin_over_eps=max((k["margin"] / k["eps"] for k in kinds),
                                              default=0.0))
        assert rel_t <= 2e-5
        assert flips == 0
    print(f"{mism_total} id mismatches in {total} rays; unexplained {unexplained[:5]}")
    assert mism_total <= int(50e-6 * total)
    assert not unexplained
