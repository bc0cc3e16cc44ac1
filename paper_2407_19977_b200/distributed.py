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


def _global_rank(group, rank: int) -> int:
    import torch.distributed as dist
    return rank if group is None else dist.get_global_rank(group, rank)


def _packed(acc):
    """One int32 buffer [sum as float32 bits (3n) | valid (n) | invalid (n)]
    on the accumulator's device, so a merge is one collective."""
    import torch
    return torch.cat([acc.sum.view(torch.int32), acc.valid, acc.invalid])


def _unpack_into(acc, buf) -> None:
    import torch
    n3 = acc.sum.numel()
    n = acc.valid.numel()
    acc.sum.copy_(buf[:n3].view(torch.float32))
    acc.valid.copy_(buf[n3:n3 + n])
    acc.invalid.copy_(buf[n3 + n:])


def merge_tiles(acc, group=None, dst: int | None = 0) -> None:
    """Merge the per-rank accumulators of a tile-sharded render: every
    element is non-zero on at most one rank (its pixel's tile owner; x + 0 =
    x), so an integer SUM of the packed buffers -- float32 bit patterns plus
    counts -- is exact.  One reduce onto group rank `dst` (its global rank
    is looked up), or one all-reduce with dst=None.  NCCL reduces CUDA
    tensors; gloo stages through host memory."""
    import torch.distributed as dist
    host_staged = dist.get_backend(group) == "gloo"
    buf = _packed(acc)
    x = buf.cpu() if (host_staged and buf.is_cuda) else buf
    if dst is None:
        dist.all_reduce(x, op=dist.ReduceOp.SUM, group=group)
    else:
        dist.reduce(x, dst=_global_rank(group, dst), op=dist.ReduceOp.SUM, group=group)
    if dst is None or dist.get_rank(group) == dst:
        _unpack_into(acc, x.to(acc.sum.device))


def merge_spp_ordered(acc, group=None, dst: int | None = 0) -> None:
    """Merge the partial accumulators of an spp-split render: gather the
    packed partials onto group rank `dst` and add them there in rank order
    (a fixed fp32 order => the same result on every run and for any
    placement of ranks); dst=None broadcasts the sum back to every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    host_staged = dist.get_backend(group) == "gloo"
    root = 0 if dst is None else dst
    buf = _packed(acc)
    x = buf.cpu() if (host_staged and buf.is_cuda) else buf
    parts = [torch.empty_like(x) for _ in range(world)] if rank == root else None
    dist.gather(x, gather_list=parts, dst=_global_rank(group, root), group=group)
    n3 = acc.sum.numel()
    if rank == root:
        total = parts[0].clone()
        tf = total[:n3].view(torch.float32)
        for p in parts[1:]:
            tf += p[:n3].view(torch.float32)
            total[n3:] += p[n3:]
        x = total
    if dst is None:
        dist.broadcast(x, src=_global_rank(group, root), group=group)
    if dst is None or rank == root:
        _unpack_into(acc, x.to(acc.sum.device))


def render_distributed(scene, settings, bvh=None, *, tile_size: int = 16, mode: str = "tiles",
                       device: int | None = None, flags: int = 0, group=None):
    """render_progressive across all ranks of `group` (default: the world):
    mode "tiles" (interleaved tiles, bit-identical to one GPU) or "spp"
    (contiguous sample ranges, for small frames / huge spp: C5).  Pass a
    DeviceScene to keep the scene resident across calls; a scene
    description is uploaded by every call, as render_progressive does.
    Returns the RenderResult on group rank 0 and None elsewhere."""
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
