"""Generate the golden fixtures by running the REFERENCE itself.

Run here (the container that holds /root/reference); the .npz outputs are
committed and travel with the repo -- nothing at test time reads
/root/reference.

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Each scene fixture stores the reference's inputs (triangles, materials,
environment, camera pack, the reference-built BVH) and outputs:
  * intersect_scene_batch / brute_force_intersect_batch / traversal counts
    on a mixed ray set (test_bvh.py:35-48 style),
  * render_progressive (accum mean, invalid counts) at a small size,
  * per-sample radiance at matched streams: `_render_pass` on zeroed
    buffers with sample_count=1 (exactly sample s of every pixel),
  * trace_radiance on explicit rays and PCG states.
Material fixtures: sample_bsdf / eval_bsdf / pdf_bsdf on random inputs.
RNG fixtures: pcg_seed / seed_stream / draws.
"""
from __future__ import annotations

import os
import sys
from pathlib import Path

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
REF = Path("/root/reference/pkg/src")
sys.path.insert(0, str(REF))
HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))

import numpy as np  # noqa: E402

import luxtrace as lx  # noqa: E402
from luxtrace.integrator import _camera_pack, _render_pass, _scene_arrays  # noqa: E402

import workloads as procgen  # noqa: E402  (scene geometry only)


def mixed_rays(n, seed, spread=1.4, radius=3.0, center=(0.0, 0.0, 0.0)):
    """Origins on an enclosing sphere aimed near the model plus a tail of
    unrelated rays (test_bvh.py:35-48)."""
    rng = np.random.default_rng(seed)
    n_aimed = int(n * 0.8)
    o = rng.normal(size=(n, 3))
    o /= np.linalg.norm(o, axis=1, keepdims=True)
    o = o * radius + np.asarray(center)
    tgt = rng.uniform(-spread, spread, size=(n, 3)) + np.asarray(center)
    d = np.empty_like(o)
    d[:n_aimed] = tgt[:n_aimed] - o[:n_aimed]
    d[n_aimed:] = rng.normal(size=(n - n_aimed, 3))
    d /= np.linalg.norm(d, axis=1, keepdims=True)
    return o, d


def to_ref_scene(scene):
    """Convert a package SceneDescription into reference objects."""
    t = scene.triangles
    tb = lx.TriangleBuffer(t.v0, t.v1, t.v2, t.n0, t.n1, t.n2, t.material_index)
    mats = [lx.OpenPbrParams(
        base_weight=m.base_weight, base_color=tuple(m.base_color),
        base_metalness=m.base_metalness, specular_weight=m.specular_weight,
        specular_color=tuple(m.specular_color), specular_roughness=m.specular_roughness,
        specular_ior=m.specular_ior, emission_luminance=m.emission_luminance,
        emission_color=tuple(m.emission_color)) for m in scene.materials]
    c = scene.camera
    cam = lx.CameraConfig(position=c.position, look_at=c.look_at, up=c.up,
                          vertical_fov_deg=c.vertical_fov_deg, width=c.width, height=c.height)
    e = scene.environment
    env = (lx.EnvironmentConfig.uniform(e.radiance) if e.kind == "uniform"
           else lx.EnvironmentConfig.gradient(e.zenith, e.horizon))
    return lx.SceneDescription(tb, mats, cam, env, 0)


def floor_scene():
    s = 50.0
    v = np.array([[-s, -s, 0.0], [s, -s, 0.0], [s, s, 0.0], [-s, s, 0.0]])
    up = np.tile([0.0, 0.0, 1.0], (2, 1))
    tb = lx.TriangleBuffer(np.array([v[0], v[0]]), np.array([v[1], v[2]]),
                           np.array([v[2], v[3]]), up, up, up)
    mat = lx.OpenPbrParams(base_color=(0.25, 0.5, 0.75), specular_weight=0.0)
    cam = lx.CameraConfig(position=(0.0, 0.0, 5.0), look_at=(0.0, 0.0, 0.0), width=16, height=16,
                          vertical_fov_deg=60.0)
    return lx.SceneDescription(tb, [mat], cam, lx.EnvironmentConfig.uniform((2.0, 2.0, 2.0)), 0)


def shell_scene():
    pos, idx = lx.icosphere(subdivisions=1)
    f = idx.reshape(-1, 3)
    c = pos[f]
    fn = np.cross(c[:, 1] - c[:, 0], c[:, 2] - c[:, 0])
    fn /= np.linalg.norm(fn, axis=1, keepdims=True)
    tb = lx.TriangleBuffer(c[:, 0], c[:, 1], c[:, 2], fn, fn, fn)
    mat = lx.OpenPbrParams(base_color=(0.5, 0.5, 0.5), specular_weight=0.0,
                           emission_luminance=0.5)
    cam = lx.CameraConfig(position=(0.0, 0.0, 0.0), look_at=(0.0, 0.0, -1.0), width=16,
                          height=16, vertical_fov_deg=90.0)
    return lx.SceneDescription(tb, [mat], cam, lx.EnvironmentConfig.uniform((0.0, 0.0, 0.0)), 0)


def glossy_scene():
    """icosphere fixture (generate.py:45-51) + icosphere_config.json."""
    pos, idx = lx.icosphere(subdivisions=2, radius=1.0)
    nrm = pos / np.linalg.norm(pos, axis=1, keepdims=True)
    pos = pos.astype(np.float32).astype(np.float64)   # GLB stores float32
    nrm = nrm.astype(np.float32).astype(np.float64)
    nrm /= np.linalg.norm(nrm, axis=1, keepdims=True)
    f = idx.reshape(-1, 3)
    tb = lx.TriangleBuffer(pos[f[:, 0]], pos[f[:, 1]], pos[f[:, 2]],
                           nrm[f[:, 0]], nrm[f[:, 1]], nrm[f[:, 2]])
    mat = lx.OpenPbrParams(base_color=(0.85, 0.7, 0.45), base_metalness=1.0,
                           specular_roughness=0.35)
    cam = lx.CameraConfig(position=(0.0, 0.6, 3.2), look_at=(0.0, 0.0, 0.0), width=32, height=24,
                          vertical_fov_deg=45.0)
    env = lx.EnvironmentConfig.gradient((0.45, 0.55, 0.85), (0.95, 0.88, 0.78))
    return lx.SceneDescription(tb, [mat], cam, env, 0)


def sphere2k_scene():
    """bumpy_sphere(2000) with mixed reference materials on a metal floor."""
    pos, idx = lx.bumpy_sphere(2000)
    f = idx.reshape(-1, 3)
    nrm = lx.generate_smooth_normals(pos, idx)
    n = f.shape[0]
    v0, v1, v2 = pos[f[:, 0]], pos[f[:, 1]], pos[f[:, 2]]
    n0, n1, n2 = nrm[f[:, 0]], nrm[f[:, 1]], nrm[f[:, 2]]
    mi = (np.arange(n) % 3).astype(np.int32)
    g = 4.0
    fv0 = np.array([[-g, -1.2, -g], [-g, -1.2, -g]])
    fv1 = np.array([[-g, -1.2, g], [g, -1.2, g]])
    fv2 = np.array([[g, -1.2, g], [g, -1.2, -g]])
    fn = np.tile([0.0, 1.0, 0.0], (2, 1))
    tb = lx.TriangleBuffer(np.vstack([v0, fv0]), np.vstack([v1, fv1]), np.vstack([v2, fv2]),
                           np.vstack([n0, fn]), np.vstack([n1, fn]), np.vstack([n2, fn]),
                           np.concatenate([mi, [3, 3]]).astype(np.int32))
    mats = [lx.OpenPbrParams(base_color=(0.8, 0.3, 0.2), specular_roughness=0.5),
            lx.OpenPbrParams(base_color=(0.9, 0.8, 0.5), base_metalness=1.0,
                             specular_roughness=0.2),
            lx.OpenPbrParams(base_color=(0.2, 0.5, 0.8), specular_weight=0.0,
                             emission_luminance=0.5, emission_color=(1.0, 0.5, 0.25)),
            lx.OpenPbrParams(base_color=(0.9, 0.9, 0.9), base_metalness=1.0,
                             specular_roughness=0.0)]
    cam = lx.CameraConfig(position=(0.0, 0.5, 3.5), look_at=(0.0, 0.0, 0.0), width=32,
                          height=24, vertical_fov_deg=45.0)
    env = lx.EnvironmentConfig.gradient((0.5, 0.6, 0.9), (0.9, 0.85, 0.8))
    return lx.SceneDescription(tb, mats, cam, env, 0)


def dup_scene():
    """test_bvh.py:125-146: an exactly duplicated triangle."""
    pos, idx = lx.bumpy_sphere(40)
    f = idx.reshape(-1, 3)
    v0, v1, v2 = pos[f[:, 0]], pos[f[:, 1]], pos[f[:, 2]]
    n = np.cross(v1 - v0, v2 - v0)
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    cat = lambda a: np.concatenate([a, a[:1]])
    tb = lx.TriangleBuffer(cat(v0), cat(v1), cat(v2), cat(n), cat(n), cat(n))
    cam = lx.CameraConfig(position=(0.0, 0.0, 3.0), look_at=(0.0, 0.0, 0.0), width=8, height=8)
    return lx.SceneDescription(tb, [lx.OpenPbrParams()], cam,
                               lx.EnvironmentConfig.uniform((1.0, 1.0, 1.0)), 0)


def mats_table(mats):
    packed = lx.pack_materials(mats)
    names = ("base_weight", "base_color", "base_metalness", "specular_weight", "specular_color",
             "specular_roughness", "specular_ior", "emission_luminance", "emission_color")
    return {f"mat_{k}": v for k, v in zip(names, packed)}


def scene_fixture(name, scene, settings, n_rays=2000, ray_radius=3.0, ray_center=(0, 0, 0),
                  spread=1.4, per_sample=4):
    bvh = lx.build_bvh(scene.triangles)
    assert lx.validate_bvh(bvh, scene.triangles) == []
    t = scene.triangles
    out = dict(v0=t.v0, v1=t.v1, v2=t.v2, n0=t.n0, n1=t.n1, n2=t.n2,
               material_index=t.material_index,
               bvh_bounds_min=bvh.bounds_min, bvh_bounds_max=bvh.bounds_max,
               bvh_left=bvh.left_child, bvh_right=bvh.right_child,
               bvh_first=bvh.first_triangle, bvh_count=bvh.triangle_count,
               bvh_order=bvh.triangle_order,
               cam_pack=_camera_pack(scene.camera),
               cam_position=scene.camera.position, cam_look_at=scene.camera.look_at,
               cam_up=scene.camera.up, cam_fov=scene.camera.vertical_fov_deg,
               width=scene.camera.width, height=scene.camera.height,
               env_kind=scene.environment.kind,
               env_radiance=scene.environment.radiance, env_zenith=scene.environment.zenith,
               env_horizon=scene.environment.horizon,
               spp=settings.samples_per_pixel, max_depth=settings.max_depth,
               rr_start=settings.rr_start_depth, seed=settings.seed, t_min=settings.t_min,
               **mats_table(scene.materials))
    # rays
    o, d = mixed_rays(n_rays, 52, spread=spread, radius=ray_radius, center=ray_center)
    out["rays_o"], out["rays_d"] = o, d
    out["isect_idx"], out["isect_t"] = lx.intersect_scene_batch(t, bvh, o, d)
    out["brute_idx"], out["brute_t"] = lx.brute_force_intersect_batch(t, o, d)
    out["count_nodes"], out["count_tests"] = lx.traversal_counts_batch(t, bvh, o, d)
    # full render
    res = lx.render_progressive(scene, settings, bvh=bvh)
    out["render_image"], out["render_invalid"] = res.image, res.invalid_samples
    # per-sample values at matched streams
    bvh_t, tri_t, mats, env_t = _scene_arrays(scene, bvh)
    cam = _camera_pack(scene.camera)
    w, h = scene.camera.width, scene.camera.height
    ps = []
    for s in range(per_sample):
        acc = np.zeros((h, w, 3))
        val = np.zeros((h, w), np.int64)
        inv = np.zeros((h, w), np.int64)
        _render_pass(acc, val, inv, s, 1, cam, w, h, *bvh_t, *tri_t, *mats, *env_t,
                     settings.seed, settings.max_depth, settings.rr_start_depth, settings.t_min)
        ps.append(np.where(val[..., None] > 0, acc, np.nan))
    out["per_sample"] = np.stack(ps)
    # trace_radiance with explicit states
    rng = np.random.default_rng(7)
    tr_rgb, tr_state, tr_in = [], [], []
    for k in range(16):
        st = (int(rng.integers(0, 2**62)), int(rng.integers(0, 2**62)) | 1)
        ray = lx.Ray(o[k], d[k])
        rad, (s_out, _) = lx.trace_radiance(scene, bvh, ray, settings, st)
        tr_rgb.append(rad)
        tr_state.append(s_out)
        tr_in.append(st)
    out["trace_rgb"] = np.array(tr_rgb)
    out["trace_state_out"] = np.array(tr_state, dtype=np.uint64)
    out["trace_state_in"] = np.array(tr_in, dtype=np.uint64)
    np.savez_compressed(HERE / f"scene_{name}.npz", **out)
    print(f"scene_{name}: {len(t)} tris, {len(bvh.left_child)} nodes, "
          f"{int((out['isect_idx'] >= 0).sum())}/{n_rays} hits")


def rng_fixture():
    out = {}
    rng = lx.pcg_seed(42, 54)
    vals = []
    for _ in range(8):
        v, rng = lx.pcg_next_u32(rng)
        vals.append(v)
    out["kat_42_54"] = np.array(vals, np.uint64)
    g = np.random.default_rng(3)
    keys = np.stack([g.integers(0, 2**31, 64), g.integers(0, 2**20, 64),
                     g.integers(0, 2**62, 64)], axis=1).astype(np.uint64)
    keys[:4] = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [12345, 678, 2**63 + 5]]
    states, draws = [], []
    for pix, smp, seed in keys.tolist():
        st = lx.seed_stream(pix, smp, seed)
        states.append((st.state, st.increment))
        row = []
        for _ in range(6):
            v, st = lx.pcg_next_u32(st)
            row.append(v)
        draws.append(row)
    out["stream_keys"] = keys
    out["stream_states"] = np.array(states, np.uint64)
    out["stream_draws"] = np.array(draws, np.uint64)
    np.savez_compressed(HERE / "rng.npz", **out)
    print("rng fixture")


def material_fixture():
    rng = np.random.default_rng(10)
    rows = []
    params = []
    for k in range(3000):
        p = lx.OpenPbrParams(
            base_weight=float(rng.uniform(0.0, 1.0)) if k % 7 else 0.0,
            base_color=tuple(rng.uniform(0.05, 1.0, 3)),
            base_metalness=float(rng.choice([0.0, 1.0, rng.uniform()])),
            specular_weight=float(rng.choice([0.0, 1.0, rng.uniform()])),
            specular_color=tuple(rng.uniform(0.2, 1.0, 3)),
            specular_roughness=float(rng.choice([0.0, 0.005, rng.uniform(), 1.0])),
            specular_ior=float(rng.uniform(1.0, 2.5)))
        n = lx.normalize(rng.normal(size=3))
        wo = lx.normalize(rng.normal(size=3))
        if np.dot(wo, n) < 0.0:
            wo = lx.normalize(wo - 2.0 * np.dot(wo, n) * n)
        if np.dot(wo, n) < 1e-4:
            continue
        u = rng.uniform(0.0, 1.0, 3)
        s = lx.sample_bsdf(wo, n, p, tuple(u))
        wi_probe = lx.normalize(rng.normal(size=3))
        f = lx.eval_bsdf(wo, wi_probe, n, p)
        pdf = lx.pdf_bsdf(wo, wi_probe, n, p)
        params.append([p.base_weight, *p.base_color, p.base_metalness, p.specular_weight,
                       *p.specular_color, p.specular_roughness, p.specular_ior])
        rows.append(np.concatenate([
            wo, n, u, [1.0 if s is not None else 0.0],
            s.direction if s is not None else np.zeros(3),
            s.throughput_weight if s is not None else np.zeros(3),
            [s.pdf if s is not None else 0.0, 1.0 if (s is not None and s.is_specular_spike) else 0.0],
            wi_probe, f, [pdf]]))
    np.savez_compressed(HERE / "material.npz", params=np.array(params), rows=np.array(rows))
    print(f"material fixture: {len(rows)} cases")


def tonemap_fixture():
    """tonemap_to_u8 (tonemap.py:59-61) on HDR values spanning both knees."""
    rng = np.random.default_rng(5)
    lin = np.concatenate([
        rng.uniform(0.0, 0.1, (2000, 3)), rng.uniform(0.0, 1.0, (4000, 3)),
        rng.exponential(2.0, (2000, 3)), rng.uniform(0.0, 50.0, (500, 3)),
        np.array([[0.0, 0.0, 0.0], [0.08, 0.08, 0.08], [0.76, 0.5, 0.2], [1.0, 1.0, 1.0]])])
    lin = lin.astype(np.float32).astype(np.float64)  # the device holds fp32 radiance
    np.savez_compressed(HERE / "tonemap.npz", linear=lin, u8=lx.tonemap_to_u8(lin),
                        neutral=lx.pbr_neutral_tonemap(lin))
    print(f"tonemap fixture: {lin.shape[0]} colors")


def main():
    if "--only" in sys.argv:
        globals()[sys.argv[sys.argv.index("--only") + 1] + "_fixture"]()
        return
    tonemap_fixture()
    rng_fixture()
    material_fixture()
    S = lx.RenderSettings
    scene_fixture("floor", floor_scene(), S(samples_per_pixel=8, max_depth=2, rr_start_depth=2))
    scene_fixture("shell", shell_scene(), S(samples_per_pixel=8, max_depth=5, rr_start_depth=5))
    scene_fixture("glossy", glossy_scene(), S(samples_per_pixel=6, max_depth=4, seed=11))
    scene_fixture("sphere2k", sphere2k_scene(), S(samples_per_pixel=4, max_depth=6, seed=3))
    scene_fixture("dup", dup_scene(), S(samples_per_pixel=2, max_depth=3, seed=1), n_rays=500)
    c1 = to_ref_scene(procgen.cornell_box(32, 32, "diffuse"))
    scene_fixture("cornell_c1", c1, S(samples_per_pixel=4, max_depth=4, rr_start_depth=3, seed=7),
                  ray_radius=3.0, ray_center=(0, 1, 0), spread=1.0)
    c2 = to_ref_scene(procgen.cornell_box(32, 32, "mixed"))
    scene_fixture("cornell_c2", c2, S(samples_per_pixel=4, max_depth=8, rr_start_depth=3, seed=7),
                  ray_radius=3.0, ray_center=(0, 1, 0), spread=1.0)
    sp = procgen.sphere_on_plane(20_000, 40, 24)
    scene_fixture("sphere20k", to_ref_scene(sp),
                  S(samples_per_pixel=2, max_depth=8, rr_start_depth=3, seed=5),
                  ray_radius=4.0, ray_center=(0, 1.1, 0), spread=1.2, per_sample=2)


if __name__ == "__main__":
    main()
