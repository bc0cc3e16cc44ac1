"""The reference's stated invariants (SPEC.md "Invariants & Properties",
/root/reference/SPEC.md:430-435) checked on the CUDA path at the sizes the
spec names:

  * Russian roulette is unbiased: furnace scene, max_depth 50, rr_start 1 vs
    roulette off, overlapping 95 % confidence intervals at 10,000 paths;
  * energy: albedo <= 1 everywhere under a uniform environment L, no pixel
    above L * (1 + 5 sigma);
  * mirror property: a metalness-1, minimum-roughness plane under the
    gradient environment reproduces the mirrored environment lookup per
    pixel within 2 % after convergence;
  * estimator at depth 1: a diffuse sphere under a uniform environment,
    direct lighting only, matches rho * L within 1 %.
"""
from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def lb():
    import paper_2407_19977_b200 as m
    return m


def sphere(n=20_000, material=0, radius=1.0, center=(0.0, 0.0, 0.0)):
    from workloads import MeshBuilder
    pos, idx = lb().bumpy_sphere(n, bump_amplitude=0.0)
    pos = np.asarray(pos) * radius + np.asarray(center)
    return MeshBuilder().add(pos, idx, material)


def per_pixel_passes(sc, settings, passes: int):
    """(passes, h*w, 3) means of `passes` independent sample ranges."""
    m = lb()
    from paper_2407_19977_b200.integrator import Accumulator, render_pass_device
    ds = m.DeviceScene(sc)
    cam = sc.camera
    spp = settings.samples_per_pixel
    out = []
    for k in range(passes):
        acc = Accumulator(cam.width, cam.height, ds.device)
        render_pass_device(ds, cam, settings, acc, k * spp, spp)
        s = acc.sum.view(-1, 3).double().cpu().numpy()
        v = acc.valid.cpu().numpy().astype(np.float64)
        out.append(s / np.maximum(v, 1)[:, None])
    return np.stack(out)


def test_roulette_unbiased_furnace():
    """SPEC: max_depth 50; rr_start 1 vs no roulette agree within
    overlapping 95 % confidence intervals at 10,000 paths.  The scene is
    the diffuse Cornell box (many interreflections, so roulette fires at
    every depth >= 1); each of the 10,000 paths is one (pixel, sample)."""
    import workloads as wl
    m = lb()
    sc = wl.cornell_box(10, 10, "diffuse")
    means, halfw = [], []
    for rr in (1, 50):
        st = m.RenderSettings(samples_per_pixel=1, max_depth=50, rr_start_depth=rr, seed=7 + rr)
        v = per_pixel_passes(sc, st, 100).mean(axis=2).ravel()   # 100 x 100 path values
        assert v.size == 10_000
        means.append(v.mean())
        halfw.append(1.96 * v.std(ddof=1) / np.sqrt(v.size))
    lo = max(means[0] - halfw[0], means[1] - halfw[1])
    hi = min(means[0] + halfw[0], means[1] + halfw[1])
    print(f"rr_start 1: {means[0]:.5f} +- {halfw[0]:.5f}; off: {means[1]:.5f} +- {halfw[1]:.5f}")
    assert lo <= hi, (means, halfw)
    assert means[1] > 0.0


def test_energy_never_exceeds_environment():
    """SPEC: albedo <= 1 everywhere and uniform environment L: no pixel
    exceeds L * (1 + 5 sigma)."""
    m = lb()
    rng = np.random.default_rng(3)
    mats = []
    for _ in range(6):
        mats.append(m.OpenPbrParams(
            base_color=tuple(rng.uniform(0.2, 1.0, 3)), base_metalness=float(rng.uniform()),
            specular_roughness=float(rng.uniform(0.0, 1.0)),
            specular_color=tuple(rng.uniform(0.5, 1.0, 3)),
            specular_ior=float(rng.uniform(1.2, 2.5))))
    mb = sphere(8_000, 0)
    for k in range(1, 6):
        c = (2.2 * np.cos(k * 1.3), 0.3 * k - 0.9, 2.2 * np.sin(k * 1.3))
        mb.parts.extend(sphere(4_000, k, 0.6, c).parts)
    L = 1.5
    cam = m.CameraConfig(position=(0, 1.5, 7), look_at=(0, 0, 0), width=48, height=36)
    sc = m.SceneDescription(mb.build(), mats, cam, m.EnvironmentConfig.uniform((L, L, L)))
    st = m.RenderSettings(samples_per_pixel=32, max_depth=12)
    p = per_pixel_passes(sc, st, 8)                        # 8 x 32 spp
    mean = p.mean(axis=0)
    sigma = p.std(axis=0, ddof=1) / np.sqrt(p.shape[0])
    assert np.all(mean <= L * (1.0 + 5.0 * sigma) + 1e-6), float((mean - L).max())


def test_mirror_plane_reflects_gradient_environment():
    """SPEC: metalness 1, minimum roughness plane under the gradient
    environment reproduces the mirrored environment lookup per pixel within
    2 % after convergence."""
    m = lb()
    from workloads import MeshBuilder, quad
    mirror = m.OpenPbrParams(base_color=(1, 1, 1), base_metalness=1.0, specular_roughness=0.0)
    g = 60.0
    mb = MeshBuilder().add_flat(quad((-g, 0, -g), (-g, 0, g), (g, 0, g), (g, 0, -g)), 0)
    W, H = 64, 48
    cam = m.CameraConfig(position=(0, 2, 4), look_at=(0, 0, 0), width=W, height=H)
    env = m.EnvironmentConfig.gradient((0.2, 0.3, 0.8), (0.9, 0.8, 0.7))
    sc = m.SceneDescription(mb.build(), [mirror], cam, env)
    img = m.render_image(sc, m.RenderSettings(samples_per_pixel=256, max_depth=4))
    # expected: the environment in the mirrored direction of each pixel's
    # rays, averaged over the pixel (a 16 x 16 grid of sub-pixel rays); the
    # vectorised camera / environment below are checked against the scalar
    # API at a few points
    c = m.camera_pack(cam)
    pos, fwd, right, up, tan_half, aspect = c[0:3], c[3:6], c[6:9], c[9:12], c[12], c[13]

    def dirs(px, py):
        sx = (2.0 * px / W - 1.0) * tan_half * aspect
        sy = (1.0 - 2.0 * py / H) * tan_half
        d = fwd[None] + sx[:, None] * right[None] + sy[:, None] * up[None]
        return d / np.linalg.norm(d, axis=1, keepdims=True)

    def env_of(d):
        t = np.clip(d[:, 1], 0.0, 1.0)[:, None]
        return np.asarray(env.horizon) + (np.asarray(env.zenith) - np.asarray(env.horizon)) * t

    for px, py, jx, jy in [(0, 0, 0.5, 0.5), (31, 20, 0.25, 0.75), (63, 47, 0.9, 0.1)]:
        ray = m.generate_camera_ray(cam, px, py, (jx, jy))
        assert np.allclose(dirs(np.array([px + jx]), np.array([py + jy]))[0], ray.direction,
                           atol=1e-12)
        rd = ray.direction * np.array([1.0, -1.0, 1.0])
        assert np.allclose(env_of(rd[None])[0], m.environment_radiance(env, rd), atol=1e-12)
    sub = (np.arange(16) + 0.5) / 16
    want = np.zeros((H * W, 3))
    xs0 = np.tile(np.arange(W), H).astype(np.float64)
    ys0 = np.repeat(np.arange(H), W).astype(np.float64)
    for sy in sub:
        for sx in sub:
            r = dirs(xs0 + sx, ys0 + sy) * np.array([1.0, -1.0, 1.0])
            want += env_of(r)
    want = want.reshape(H, W, 3)
    want /= 256
    rel = np.abs(img - want) / want
    assert rel.max() <= 0.02, float(rel.max())


def test_depth_one_estimator_diffuse_sphere():
    """SPEC: direct-lighting-only render (one bounce) of a diffuse sphere
    under a uniform environment matches rho * L within 1 %."""
    m = lb()
    rho, L = 0.6, 2.0
    lam = m.OpenPbrParams(base_color=(rho, rho, rho), specular_weight=0.0)
    cam = m.CameraConfig(position=(0, 0, 4), look_at=(0, 0, 0), width=10, height=10,
                         vertical_fov_deg=10.0)
    sc = m.SceneDescription(sphere().build(), [lam], cam, m.EnvironmentConfig.uniform((L, L, L)))
    img = m.render_image(sc, m.RenderSettings(samples_per_pixel=64, max_depth=2))
    # every sample that leaves the surface sees L; one whose cosine sample
    # about the interpolated shading normal points into the faceted surface
    # is lost (the visibility weighting): the image mean within 1 %, no
    # pixel more than 2 % off
    assert abs(img.mean() / (rho * L) - 1.0) <= 0.01, float(img.mean())
    assert np.allclose(img, rho * L, rtol=0.02), (float(img.min()), float(img.max()))
