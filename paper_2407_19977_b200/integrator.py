"""The north-star path: progressive Monte-Carlo rendering on the GPU.

Drop-in for luxtrace.integrator (integrator.py:41-356): same names,
arguments, result type and error behaviour.  Every sample is computed by the
sm_100a wavefront kernels behind lt_render_pass (raygen -> closest-hit
traversal -> OpenPBR shade/RR/compaction -> ordered accumulation), keyed by
the reference's per-(pixel, sample) PCG32 streams.  There is no CPU path.

Differences from the reference, all deliberate:
  * RenderSettings accepts rr_start_depth > max_depth (roulette simply never
    triggers), which the reference's own tests rely on;
  * `threads` is accepted and has no effect on the GPU render (reported
    back as the clamped host worker count, as the reference reports it);
  * per-sample arithmetic is fp32 (tolerances in tests/), accumulation is an
    fp32 per-pixel sum in sample order, returned as a float64 mean.
"""
from __future__ import annotations

import ctypes as C
import math
import time
import warnings
from dataclasses import dataclass

import numpy as np

from . import _lib
from .device import DeviceScene
from .geometry import DEFAULT_T_MIN, Ray
from .scene import camera_pack, environment_pack

RR_MIN_SURVIVAL = 0.05                 # integrator.py:34
INVALID_SAMPLE_WARN_FRACTION = 1e-4    # integrator.py:35


@dataclass(frozen=True)
class RenderSettings:
    samples_per_pixel: int = 100
    max_depth: int = 5
    rr_start_depth: int = 3
    seed: int = 0
    t_min: float = DEFAULT_T_MIN

    def __post_init__(self) -> None:
        if self.samples_per_pixel < 1:
            raise ValueError("samples_per_pixel must be >= 1")
        if self.max_depth < 1:
            raise ValueError("max_depth must be >= 1")
        if self.rr_start_depth < 0:
            raise ValueError("rr_start_depth must be >= 0")
        if self.seed < 0:
            raise ValueError("seed must be non-negative")
        if not self.t_min > 0.0:
            raise ValueError("t_min must be positive")


@dataclass
class RenderResult:
    image: np.ndarray                 # (h, w, 3) float64 linear radiance means
    samples_per_pixel: int
    invalid_samples: np.ndarray       # (h, w) int64 non-finite estimates dropped
    elapsed_ms: float
    threads_used: int


def render_params(camera, settings, sample_start: int, sample_count: int, *, flags: int = 0,
                  shard=None, max_batch_paths: int = 0) -> _lib.RenderParams:
    p = _lib.RenderParams()
    p.camera[:] = [float(x) for x in camera_pack(camera)]
    p.width, p.height = int(camera.width), int(camera.height)
    p.sample_start, p.sample_count = int(sample_start), int(sample_count)
    p.seed = int(settings.seed) & ((1 << 64) - 1)
    p.max_depth, p.rr_start = int(settings.max_depth), int(settings.rr_start_depth)
    p.t_min = float(settings.t_min)
    if shard is not None:
        rank, n_ranks, tile = shard
        p.rank, p.n_ranks, p.tile_size = int(rank), int(n_ranks), int(tile)
    else:
        p.rank, p.n_ranks, p.tile_size = 0, 1, 1
    p.flags = int(flags)
    p.max_batch_paths = int(max_batch_paths)
    return p


class Accumulator:
    """Device accumulation buffers of one image: per-pixel fp32 RGB sum and
    valid / invalid sample counts (torch tensors on the scene's GPU)."""

    def __init__(self, width: int, height: int, device: int):
        import torch
        self.width, self.height = int(width), int(height)
        self.device = torch.device("cuda", device)
        n = self.width * self.height
        self.sum = torch.zeros(n * 3, dtype=torch.float32, device=self.device)
        self.valid = torch.zeros(n, dtype=torch.int32, device=self.device)
        self.invalid = torch.zeros(n, dtype=torch.int32, device=self.device)

    def pointers(self):
        return (C.c_void_p(self.sum.data_ptr()), C.c_void_p(self.valid.data_ptr()),
                C.c_void_p(self.invalid.data_ptr()))

    def mean(self):
        """(h, w, 3) float64 device tensor: sum / valid (0 where no sample)."""
        h, w = self.height, self.width
        v = self.valid.view(h, w, 1).clamp_min(1).double()
        return self.sum.view(h, w, 3).double() / v


def render_pass_device(ds: DeviceScene, camera, settings, acc: Accumulator, sample_start: int,
                       sample_count: int, *, flags: int = 0, shard=None,
                       max_batch_paths: int = 0, stream=None) -> None:
    """One `_render_pass` (integrator.py:230-277) into device buffers."""
    import torch
    p = render_params(camera, settings, sample_start, sample_count, flags=flags, shard=shard,
                      max_batch_paths=max_batch_paths)
    st = stream if stream is not None else torch.cuda.current_stream(acc.device)
    _lib.check(_lib.lib().lt_render_pass(ds.handle, C.byref(p), *acc.pointers(),
                                         C.c_void_p(st.cuda_stream)))


def render_pass(scene, accum, valid_count, invalid_count, sample_start: int, sample_count: int,
                settings, camera=None, *, flags: int = 0, shard=None) -> None:
    """Host-buffer drop-in for `_render_pass`: updates the (h, w, 3) float64
    running means and (h, w) int64 counts in place with samples
    [sample_start, sample_start + sample_count)."""
    ds = scene if isinstance(scene, DeviceScene) else DeviceScene(scene)
    cam = camera if camera is not None else ds.camera
    for name, a, dt in (("accum", accum, np.float64), ("valid_count", valid_count, np.int64),
                        ("invalid_count", invalid_count, np.int64)):
        if a.dtype != dt or not a.flags.c_contiguous:
            raise ValueError(f"{name} must be a C-contiguous {np.dtype(dt).name} array")
    if accum.shape != (cam.height, cam.width, 3):
        raise ValueError("accum shape does not match the camera")
    p = render_params(cam, settings, sample_start, sample_count, flags=flags, shard=shard)
    P = _lib.ptr
    _lib.check(_lib.lib().lt_render_pass_host(ds.handle, C.byref(p), P(accum, C.c_double),
                                              P(valid_count, C.c_int64),
                                              P(invalid_count, C.c_int64)))


def render_progressive(scene, settings: RenderSettings, bvh=None, threads: int | None = None,
                       progress=None, progress_interval: int = 1, *, device: int | None = None,
                       flags: int = 0, shard=None, max_batch_paths: int = 0,
                       return_device: bool = False) -> RenderResult:
    """Render the full sample budget (integrator.py:310-350).  With a
    `progress` callback the image advances `progress_interval` samples at a
    time and `progress(samples_done, elapsed_ms)` runs after each chunk;
    chunking never changes the result (samples accumulate in index order)."""
    import torch
    if device is None:
        device = scene.device if isinstance(scene, DeviceScene) else 0
    owned = not isinstance(scene, DeviceScene)
    t_scene = time.perf_counter()
    ds = DeviceScene(scene, bvh, device=device) if owned else scene
    scene_wall_ms = (time.perf_counter() - t_scene) * 1e3
    cam = ds.camera
    acc = Accumulator(cam.width, cam.height, ds.device)
    st = torch.cuda.current_stream(acc.device)
    spp = settings.samples_per_pixel
    chunk = max(1, int(progress_interval)) if progress is not None else spp
    start = time.perf_counter()
    done = 0
    while done < spp:
        step = min(chunk, spp - done)
        render_pass_device(ds, cam, settings, acc, done, step, flags=flags, shard=shard,
                           max_batch_paths=max_batch_paths, stream=st)
        done += step
        if progress is not None:
            st.synchronize()
            progress(done, (time.perf_counter() - start) * 1000.0)
    st.synchronize()
    elapsed_ms = (time.perf_counter() - start) * 1000.0
    if return_device:
        return acc
    t0 = time.perf_counter()
    image, invalid = fetch_image(acc, st)
    d2h_ms = (time.perf_counter() - t0) * 1e3
    dropped = int(invalid.sum())
    total = spp * cam.width * cam.height
    if dropped > total * INVALID_SAMPLE_WARN_FRACTION:
        warnings.warn(f"{dropped} of {total} samples were non-finite and dropped",
                      RuntimeWarning, stacklevel=2)
    # `threads` keeps its meaning as the host worker count (clamped as the
    # reference clamps it, _parallel.py:27-36); the GPU render ignores it
    from ._parallel import set_worker_count
    res = RenderResult(image, spp, invalid, elapsed_ms, set_worker_count(threads))
    res.timings = {"scene_create_ms": ds.create_ms if owned else 0.0,
                   "scene_wall_ms": scene_wall_ms if owned else 0.0, "render_ms": elapsed_ms,
                   "image_d2h_ms": d2h_ms}
    if owned:
        t0 = time.perf_counter()
        ds.close()
        res.timings["scene_release_ms"] = (time.perf_counter() - t0) * 1e3
    return res


_PINNED_PRIMED: set = set()


def fetch_image(acc: Accumulator, stream=None):
    """(h, w, 3) float64 means and (h, w) int64 invalid counts on the host.
    Both are produced in their final dtype on the device and copied once into
    page-locked buffers from torch's caching host allocator; the returned
    arrays own those buffers (no host-side copy), which return to the cache
    when the caller drops them."""
    import torch
    h, w = acc.height, acc.width
    key = (h, w)
    if key not in _PINNED_PRIMED:
        # page-locking is slow (tens of ms for a 1080p result); two spare
        # pairs stay in the allocator's cache so a caller that still holds the
        # previous image (res = render(...) in a loop) never pins anew
        spare = [(torch.empty((h, w, 3), dtype=torch.float64, pin_memory=True),
                  torch.empty((h, w), dtype=torch.int64, pin_memory=True)) for _ in range(2)]
        del spare
        _PINNED_PRIMED.add(key)
    mean_h = torch.empty((h, w, 3), dtype=torch.float64, pin_memory=True)
    inv_h = torch.empty((h, w), dtype=torch.int64, pin_memory=True)
    st = stream or torch.cuda.current_stream(acc.device)
    mean_d = torch.empty((h, w, 3), dtype=torch.float64, device=acc.device)
    inv_d = torch.empty((h, w), dtype=torch.int64, device=acc.device)
    # sum / max(valid, 1) and the int64 counts in one launch (Accumulator.mean's
    # arithmetic), then one copy each
    _lib.check(_lib.lib().lt_accum_finish(*acc.pointers(), h * w, C.c_void_p(mean_d.data_ptr()),
                                          C.c_void_p(inv_d.data_ptr()),
                                          C.c_void_p(st.cuda_stream)))
    mean_h.copy_(mean_d, non_blocking=True)
    inv_h.copy_(inv_d, non_blocking=True)
    st.synchronize()
    return mean_h.numpy(), inv_h.numpy()


def render_image(scene, settings: RenderSettings, bvh=None, threads: int | None = None,
                 **kw) -> np.ndarray:
    return render_progressive(scene, settings, bvh=bvh, threads=threads, **kw).image


def trace_radiance_batch(scene, bvh, origins, directions, settings, states, incs, *,
                         device: int = 0):
    """Many independent paths with caller-supplied PCG (state, increment);
    returns (rgb (n, 3) float64, advanced states (n,) uint64)."""
    ds = scene if isinstance(scene, DeviceScene) else DeviceScene(scene, bvh, device=device)
    o = np.ascontiguousarray(origins, dtype=np.float64).reshape(-1, 3)
    d = np.ascontiguousarray(directions, dtype=np.float64).reshape(-1, 3)
    s = np.ascontiguousarray(states, dtype=np.uint64).reshape(-1)
    c = np.ascontiguousarray(incs, dtype=np.uint64).reshape(-1)
    n = o.shape[0]
    if d.shape != o.shape or s.shape != (n,) or c.shape != (n,):
        raise ValueError("origins, directions, states and increments must agree in length")
    rgb = np.zeros((n, 3))
    out = np.zeros(n, np.uint64)
    if n:
        P = _lib.ptr
        _lib.check(_lib.lib().lt_trace_paths_host(
            ds.handle, P(o, C.c_double), P(d, C.c_double), P(s, C.c_uint64), P(c, C.c_uint64),
            n, int(settings.max_depth), int(settings.rr_start_depth), float(settings.t_min),
            P(rgb, C.c_double), P(out, C.c_uint64)))
    return rgb, out


def trace_radiance(scene, bvh, ray: Ray, settings: RenderSettings,
                   rng_state: tuple[int, int]):
    """One path for one explicit ray (integrator.py:294-307).  Returns
    (radiance, (advanced state, increment))."""
    rgb, out = trace_radiance_batch(scene, bvh, ray.origin[None], ray.direction[None], settings,
                                    [int(rng_state[0]) & ((1 << 64) - 1)],
                                    [int(rng_state[1]) & ((1 << 64) - 1)])
    return rgb[0], (int(out[0]), int(rng_state[1]))


def _camera_dir(cam, px, py, jx, jy, width, height):
    """_camera_dir (integrator.py:86-98) in Python floats (host API only)."""
    sx = 2.0 * (px + jx) / width - 1.0
    sy = 1.0 - 2.0 * (py + jy) / height
    hx = cam[12] * cam[13] * sx
    hy = cam[12] * sy
    dx = cam[3] + cam[6] * hx + cam[9] * hy
    dy = cam[4] + cam[7] * hx + cam[10] * hy
    dz = cam[5] + cam[8] * hx + cam[11] * hy
    inv = 1.0 / math.sqrt(dx * dx + dy * dy + dz * dz)
    return dx * inv, dy * inv, dz * inv


def generate_camera_ray(camera, px: int, py: int, jitter=(0.5, 0.5)) -> Ray:
    if not (0 <= px < camera.width and 0 <= py < camera.height):
        raise ValueError(f"pixel ({px}, {py}) outside a {camera.width}x{camera.height} image")
    cam = camera_pack(camera)
    d = _camera_dir(cam, px, py, float(jitter[0]), float(jitter[1]), camera.width,
                    camera.height)
    return Ray(np.asarray(camera.position, dtype=np.float64).copy(), np.array(d))


def environment_radiance(env, direction) -> np.ndarray:
    """Host evaluation of the uniform / gradient environment (integrator.py:
    124-142)."""
    d = np.asarray(direction, dtype=np.float64)
    kind, a, b = environment_pack(env)
    if kind == 0:
        return a.copy()
    if kind == 1:
        t = min(max(float(d[1]), 0.0), 1.0)
        return b + (a - b) * t
    raise ValueError("environment_radiance is host-only for uniform/gradient environments")
