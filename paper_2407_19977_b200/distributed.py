"""Multi-GPU rendering: one process per GPU, the scene replicated in every
GPU's HBM, the image sharded by interleaved tiles, partial accumulators
merged over NCCL (torch.distributed) -- SURVEY §8(e).

Tile sharding: square tiles of `tile_size` in raster order, tile k rendered
by rank k % world.  RNG streams stay keyed by the global pixel index, so
every pixel gets exactly the samples it would get on one GPU and the merged
accumulator (a sum of zero-padded frames; x + 0 = x) is bit-identical to the
single-GPU result.  spp splitting (rank r renders a contiguous sample range)
is the alternative for small frames; its partial sums are gathered and
added in rank order, deterministic but not bit-identical to 1 GPU because
the fp32 additions regroup.
"""
from __future__ import annotations

import numpy as np


def tile_pixels(width: int, height: int, tile: int, rank: int, world: int) -> np.ndarray:
    """Global pixel indices of `rank` (mirror of pixel_set in csrc/lt_api.cu)."""
    if world <= 1:
        return np.arange(width * height, dtype=np.int64)
    ntx = -(-width // tile)
    nty = -(-height // tile)
    out = []
    for k in range(rank, ntx * nty, world):
        ty, tx = divmod(k, ntx)
        ys = np.arange(ty * tile, min(height, (ty + 1) * tile))
        xs = np.arange(tx * tile, min(width, (tx + 1) * tile))
        out.append((ys[:, None] * width + xs[None, :]).ravel())
    return np.concatenate(out) if out else np.zeros(0, np.int64)


def spp_range(spp: int, rank: int, world: int) -> tuple[int, int]:
    """[start, stop) of rank's contiguous sample range for spp splitting."""
    lo = spp * rank // world
    hi = spp * (rank + 1) // world
    return lo, hi


def merge_tiles(acc, group=None, dst: int | None = 0) -> None:
    """Sum the zero-padded per-rank accumulators (tile sharding: exact).
    dst=None all-reduces; otherwise reduces onto rank dst.  Works for NCCL
    (CUDA tensors) and gloo (CPU tensors)."""
    import torch.distributed as dist
    host_staged = dist.get_backend(group) == "gloo"   # gloo: reduce host copies
    for t in (acc.sum, acc.valid, acc.invalid):
        x = t.cpu() if (host_staged and t.is_cuda) else t
        if dst is None:
            dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group)
        else:
            dist.reduce(x, dst=dst, op=dist.ReduceOp.SUM, group=group)
        if x is not t:
            t.copy_(x)


def merge_spp_ordered(acc, group=None) -> None:
    """spp splitting: all-gather the partial sums and add them in rank order
    on every rank (fixed fp32 order => identical result on every run)."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    host_staged = dist.get_backend(group) == "gloo"
    for t in (acc.sum, acc.valid, acc.invalid):
        x = t.cpu() if (host_staged and t.is_cuda) else t
        parts = [torch.empty_like(x) for _ in range(world)]
        dist.all_gather(parts, x, group=group)
        total = parts[0].clone()
        for p in parts[1:]:
            total += p
        t.copy_(total)


def render_distributed(scene, settings, bvh=None, *, tile_size: int = 16, mode: str = "tiles",
                       device: int | None = None, flags: int = 0, group=None):
    """render_progressive across all ranks of the default process group.
    Returns the RenderResult on rank 0 and None elsewhere."""
    import time

    import torch
    import torch.distributed as dist

    from .device import DeviceScene
    from .integrator import Accumulator, RenderResult, render_pass_device
    rank, world = dist.get_rank(group), dist.get_world_size(group)
    if device is None:
        device = torch.cuda.current_device()
    ds = scene if isinstance(scene, DeviceScene) else DeviceScene(scene, bvh, device=device)
    cam = ds.camera
    acc = Accumulator(cam.width, cam.height, ds.device)
    t0 = time.perf_counter()
    if mode == "tiles":
        render_pass_device(ds, cam, settings, acc, 0, settings.samples_per_pixel, flags=flags,
                           shard=(rank, world, tile_size))
        merge_tiles(acc, group, dst=0)
    elif mode == "spp":
        lo, hi = spp_range(settings.samples_per_pixel, rank, world)
        render_pass_device(ds, cam, settings, acc, lo, hi - lo, flags=flags)
        merge_spp_ordered(acc, group)
    else:
        raise ValueError(f"unknown sharding mode {mode!r}")
    torch.cuda.synchronize(ds.device)
    elapsed = (time.perf_counter() - t0) * 1e3
    if rank != 0:
        return None
    from .integrator import fetch_image
    image, invalid = fetch_image(acc)
    return RenderResult(image, settings.samples_per_pixel, invalid, elapsed, world)
