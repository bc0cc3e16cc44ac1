"""Host-side API mirror: types, validation and error behaviour of the
reference interface, the camera pack, the PCG API and procedural scenes.
No GPU needed; the compute entry points must refuse to run without one."""
from __future__ import annotations

import numpy as np
import pytest

import workloads as wl

from conftest import GOLDEN, golden_scene, gpu_available

import paper_2407_19977_b200 as lb


def test_settings_validation():
    with pytest.raises(ValueError):
        lb.RenderSettings(samples_per_pixel=0)
    with pytest.raises(ValueError):
        lb.RenderSettings(max_depth=0)
    with pytest.raises(ValueError):
        lb.RenderSettings(seed=-1)
    with pytest.raises(ValueError):
        lb.RenderSettings(t_min=0.0)
    with pytest.raises(ValueError):
        lb.RenderSettings(rr_start_depth=-1)
    # accepted (the reference rejects it, but its own tests rely on it)
    lb.RenderSettings(max_depth=1)


def test_material_validation():
    with pytest.raises(ValueError):
        lb.OpenPbrParams(base_weight=1.5)
    with pytest.raises(ValueError):
        lb.OpenPbrParams(base_color=(0.2, -0.1, 0.3))
    with pytest.raises(ValueError):
        lb.OpenPbrParams(specular_ior=0.9)
    with pytest.raises(ValueError):
        lb.OpenPbrParams(emission_luminance=-1.0)
    with pytest.raises(ValueError):
        lb.OpenPbrParams(coat_weight=2.0)
    t = lb.pack_material_table([lb.OpenPbrParams(), lb.OpenPbrParams(coat_weight=0.5)])
    assert t["coat_weight"].tolist() == [0.0, 0.5]
    assert t["base_color"].shape == (2, 3)


def test_camera_and_environment_validation():
    with pytest.raises(lb.SceneError):
        lb.CameraConfig(position=(0, 0, 0), look_at=(0, 0, 0))
    with pytest.raises(lb.SceneError):
        lb.CameraConfig(position=(0, 0, 0), look_at=(0, 1, 0), up=(0, 1, 0))
    with pytest.raises(lb.SceneError):
        lb.EnvironmentConfig(kind="sky")
    with pytest.raises(lb.SceneError):
        lb.EnvironmentConfig.latlong(np.zeros((4, 8)))
    env = lb.EnvironmentConfig.latlong(wl.synthetic_hdr(64, 32), 2.0)
    assert env.texels.dtype == np.float32 and env.texels.shape == (32, 64, 3)


@pytest.mark.parametrize("name", ["floor", "glossy", "cornell_c2"])
def test_camera_pack_matches_reference(name):
    g = golden_scene(name)
    assert np.array_equal(lb.camera_pack(g.camera), g["cam_pack"])


def test_pcg_api_matches_reference():
    z = np.load(GOLDEN / "rng.npz")
    rng = lb.pcg_seed(42, 54)
    out = []
    for _ in range(8):
        v, rng = lb.pcg_next_u32(rng)
        out.append(v)
    assert out == z["kat_42_54"].tolist()
    for (pix, smp, seed), (gs, gi) in zip(z["stream_keys"].tolist(), z["stream_states"].tolist()):
        s = lb.seed_stream(pix, smp, seed)
        assert (s.state, s.increment) == (gs, gi)
    u, _ = lb.next_unit_real(lb.pcg_seed(42, 54))
    assert u == out[0] / 2.0**32
    with pytest.raises(ValueError):
        lb.seed_stream(-1, 0, 0)


def test_camera_ray_geometry():
    cam = lb.CameraConfig(position=(1.0, 2.0, 3.0), look_at=(-2.0, 0.5, -1.0), width=9, height=9,
                          vertical_fov_deg=47.0)
    ray = lb.generate_camera_ray(cam, 4, 4)
    expected = lb.normalize(np.array([-2.0, 0.5, -1.0]) - np.array([1.0, 2.0, 3.0]))
    assert np.allclose(ray.direction, expected, atol=1e-12)
    with pytest.raises(ValueError, match="outside"):
        lb.generate_camera_ray(cam, 9, 0)


def test_environment_radiance_host():
    env = lb.EnvironmentConfig.gradient(zenith=(0.0, 0.0, 1.0), horizon=(1.0, 1.0, 0.0))
    assert np.allclose(lb.environment_radiance(env, (0, 1, 0)), (0, 0, 1))
    assert np.allclose(lb.environment_radiance(env, (0, -1, 0)), (1, 1, 0))


def test_bumpy_sphere_matches_reference_generator():
    g = golden_scene("sphere2k")
    pos, idx = lb.bumpy_sphere(2000)
    f = idx.reshape(-1, 3)
    assert np.array_equal(pos[f[:, 0]], g["v0"][:2000])
    assert np.array_equal(pos[f[:, 2]], g["v2"][:2000])


def test_procedural_scenes():
    c1 = wl.cornell_box(64, 64, "diffuse")
    assert 30 <= len(c1.triangles) <= 40
    # dyadic coordinates: exact in float32
    for k in ("v0", "v1", "v2"):
        a = getattr(c1.triangles, k)
        assert np.array_equal(a.astype(np.float32).astype(np.float64), a)
    ext = wl.cornell_box(32, 32, "extended")
    assert any(m.transmission_weight > 0 for m in ext.materials)
    assert any(m.coat_weight > 0 for m in ext.materials)
    pb = wl.pushbutton(64, 36, detail=0.2)
    assert len(pb.triangles) > 10_000
    assert pb.environment.kind == "latlong"


@pytest.mark.skipif(gpu_available(), reason="checks the no-GPU failure mode")
def test_compute_refuses_without_gpu():
    g = golden_scene("floor")
    with pytest.raises(RuntimeError):
        lb.render_image(g.scene, g.settings)
    with pytest.raises(RuntimeError):
        lb.intersect_scene_batch(g.triangles, g.bvh, g["rays_o"], g["rays_d"])


REFERENCE_ALL = [   # luxtrace/__init__.py:40-65
    "Aabb", "Hit", "Ray", "Triangle", "TriangleBuffer", "aabb_surface_area", "aabb_union",
    "normalize", "ray_aabb_intersect", "ray_triangle_intersect", "triangle_bounds", "vec3",
    "PcgState", "next_unit_real", "pcg_next_u32", "pcg_seed", "seed_stream",
    "BuildStats", "Bvh", "brute_force_intersect_batch", "build_bvh", "intersect_any",
    "intersect_scene", "intersect_scene_batch", "intersect_scene_counted",
    "traversal_counts_batch", "validate_bvh",
    "BsdfSample", "OpenPbrParams", "cosine_sample_hemisphere", "emitted_radiance", "eval_bsdf",
    "fresnel_schlick", "ggx_ndf", "ggx_sample_half_vector", "pack_materials", "pdf_bsdf",
    "sample_bsdf", "smith_g2",
    "CameraConfig", "EnvironmentConfig", "MaterialMap", "RenderConfig", "SceneDescription",
    "SceneError", "flatten_scene", "generate_smooth_normals", "load_gltf", "load_render_config",
    "load_scene",
    "RenderResult", "RenderSettings", "environment_radiance", "generate_camera_ray",
    "render_image", "render_progressive", "trace_radiance",
    "linear_to_srgb", "pbr_neutral_tonemap", "quantize_to_u8", "srgb_to_linear",
    "tonemap_to_u8", "write_linear_dump", "write_png",
    "bumpy_sphere", "bumpy_sphere_glb", "icosphere", "icosphere_glb", "save_glb",
    "set_worker_count", "thread_cap",
    "BenchRow", "BenchmarkReport", "auto_framing_camera", "format_ms", "load_benchmark_scene",
    "run_benchmark", "summarize_runs",
]


def test_reference_api_names_exported():
    missing = [n for n in REFERENCE_ALL if not hasattr(lb, n)]
    assert missing == []


def test_validate_bvh_flags_faults():
    """bvh.py:305-352 with the fault injections of test_bvh.py:149-174."""
    import copy
    g = golden_scene("sphere2k")
    assert lb.validate_bvh(g.bvh, g.triangles) == []
    b = copy.deepcopy(g.bvh)
    c = (b.bounds_min[0] + b.bounds_max[0]) / 2.0
    b.bounds_min = b.bounds_min.copy()
    b.bounds_max = b.bounds_max.copy()
    b.bounds_min[0], b.bounds_max[0] = c - 1e-4, c + 1e-4
    assert any("node 0" in m and "exceed" in m for m in lb.validate_bvh(b, g.triangles))
    b = copy.deepcopy(g.bvh)
    b.triangle_order = b.triangle_order.copy()
    b.triangle_order[0] = b.triangle_order[1]
    assert any("permutation" in m for m in lb.validate_bvh(b, g.triangles))
    b = copy.deepcopy(g.bvh)
    victim = int(np.nonzero(b.triangle_count > 0)[0][3])
    b.first_triangle = b.first_triangle.copy()
    b.first_triangle[victim] = len(g.triangles)
    assert any(f"node {victim}" in m and "out of bounds" in m
               for m in lb.validate_bvh(b, g.triangles))


def test_writers_and_geometry_helpers(tmp_path):
    img = (np.arange(4 * 5 * 3) % 256).astype(np.uint8).reshape(4, 5, 3)
    lb.write_png(tmp_path / "a.png", img)
    from PIL import Image
    assert np.array_equal(np.asarray(Image.open(tmp_path / "a.png")), img)
    with pytest.raises(ValueError):
        lb.write_png(tmp_path / "b.png", img.astype(np.float32))
    lin = np.linspace(0, 2, 4 * 5 * 3).reshape(4, 5, 3)
    lb.write_linear_dump(tmp_path / "a.raw", lin)
    assert np.array_equal(np.fromfile(tmp_path / "a.raw", dtype="<f4"),
                          lin.astype("<f4").ravel())
    t = lb.Triangle(lb.vec3(0, 0, 0), lb.vec3(1, 0, 0), lb.vec3(0, 2, 0), *[lb.vec3(0, 0, 1)] * 3)
    box = lb.triangle_bounds(t)
    assert np.allclose(box.min, -2e-7) and np.allclose(box.max, [1 + 2e-7, 2 + 2e-7, 2e-7])
    u = lb.aabb_union(box, lb.Aabb(lb.vec3(-1, -1, -1), lb.vec3(0, 0, 0)))
    assert np.allclose(u.min, -1.0) and lb.aabb_surface_area(lb.Aabb.empty()) == 0.0
    assert lb.set_worker_count(1) == 1 and lb.thread_cap() >= 1
