"""Multi-process host logic of the sharded render (world size 2, gloo, CPU).

Each rank computes the accumulator of its own interleaved tiles (the oracle
stands in for the per-GPU kernels, which need a device), then the merge in
paper_2407_19977_b200.distributed reduces them; the merged frame must equal
the single-process render bit for bit, and every pixel must belong to
exactly one rank.  The spp-split merge is checked for rank-order
determinism."""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_19977_b200.distributed import spp_range, tile_pixels


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class CpuAcc:
    """Accumulator-shaped CPU tensors (sum, valid, invalid)."""

    def __init__(self, n):
        self.sum = torch.zeros(n * 3, dtype=torch.float32)
        self.valid = torch.zeros(n, dtype=torch.int32)
        self.invalid = torch.zeros(n, dtype=torch.int32)


def _partial(rank, world, mode, spp, w, h):
    """This rank's accumulator, built from oracle per-sample values in
    sample order (fp32 sum, like k_accumulate)."""
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
    from conftest import golden_scene
    g = golden_scene("glossy")
    oc = g.oracle()
    acc = CpuAcc(w * h)
    if mode == "tiles":
        pix = tile_pixels(w, h, 5, rank, world)
        samples = range(spp)
    else:
        pix = np.arange(w * h)
        lo, hi = spp_range(spp, rank, world)
        samples = range(lo, hi)
    s = acc.sum.view(-1, 3).numpy()
    v = acc.valid.numpy()
    for smp in samples:
        rgb, _ = oc.sample_values(pix, smp, g["cam_pack"], w, h, 11, 4, 3, threads=1)
        rgb = rgb.astype(np.float32)
        s[pix] = s[pix] + rgb
        v[pix] += 1
    return acc


def _worker(rank, world, port, mode, spp, w, h, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_19977_b200.distributed import merge_spp_ordered, merge_tiles
    acc = _partial(rank, world, mode, spp, w, h)
    if mode == "tiles":
        merge_tiles(acc, dst=0)
    else:
        merge_spp_ordered(acc)
    if rank == 0:
        out.put((acc.sum.numpy().copy(), acc.valid.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def _run(mode, spp=4, world=2):
    g_w, g_h = 32, 24
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, spp, g_w, g_h, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3, 4])
def test_tiles_partition_the_frame(world):
    for w, h, t in ((32, 24, 5), (1920, 1080, 16), (7, 3, 4)):
        parts = [tile_pixels(w, h, t, r, world) for r in range(world)]
        allp = np.concatenate(parts)
        assert allp.size == w * h
        assert np.array_equal(np.sort(allp), np.arange(w * h))


def test_spp_ranges_cover_samples():
    for spp, world in ((256, 8), (7, 3), (2, 4)):
        rs = [spp_range(spp, r, world) for r in range(world)]
        assert rs[0][0] == 0 and rs[-1][1] == spp
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))


def test_tile_merge_is_bit_exact_gloo():
    s_merged, v_merged = _run("tiles")
    single = _partial(0, 1, "tiles", 4, 32, 24)
    assert np.array_equal(s_merged, single.sum.numpy())
    assert np.array_equal(v_merged, single.valid.numpy())


def test_spp_merge_is_deterministic_gloo():
    a = _run("spp")
    b = _run("spp")
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    single = _partial(0, 1, "spp", 4, 32, 24)
    assert np.array_equal(a[1], single.valid.numpy())
    assert np.allclose(a[0], single.sum.numpy(), rtol=1e-6, atol=1e-6)


def _subgroup_worker(rank, world, port, out):
    """World of 3; ranks {1, 2} form a group that renders the frame as a
    2-way tile split and merges onto the GROUP's rank 0 (= global rank 1)."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2407_19977_b200.distributed import merge_spp_ordered, merge_tiles
    group = dist.new_group([1, 2])
    if rank in (1, 2):
        g_rank = dist.get_rank(group)
        acc = _partial(g_rank, 2, "tiles", 3, 32, 24)
        merge_tiles(acc, group, dst=0)
        if rank == 1:
            out.put(("tiles", acc.sum.numpy().copy(), acc.valid.numpy().copy()))
        acc2 = _partial(g_rank, 2, "spp", 3, 32, 24)
        merge_spp_ordered(acc2, group, dst=None)   # every group rank gets the sum
        out.put((f"spp{rank}", acc2.sum.numpy().copy(), acc2.valid.numpy().copy()))
    dist.barrier()
    dist.destroy_process_group()


def test_merges_on_a_subgroup_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_subgroup_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = dict((k, (s, v)) for k, s, v in (q.get(timeout=120) for _ in range(3)))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    single = _partial(0, 1, "tiles", 3, 32, 24)
    assert np.array_equal(got["tiles"][0], single.sum.numpy())
    assert np.array_equal(got["tiles"][1], single.valid.numpy())
    assert np.array_equal(got["spp1"][0], got["spp2"][0])
    assert np.array_equal(got["spp1"][1], single.valid.numpy())
