"""The NCCL side of the multi-GPU path on one B200: a world-size-1 NCCL
process group runs render_distributed's CUDA-tensor collectives (the reduce
of the zero-padded tile accumulators, the rank-ordered all-gather of spp
splitting) and must reproduce render_progressive exactly.  (The N > 1 merge
logic runs under gloo on CPU in tests/test_distributed_gloo.py.)"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest

from conftest import golden_scene

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.fixture
def nccl_group():
    import torch
    import torch.distributed as dist
    os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
    os.environ["MASTER_PORT"] = str(_free_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist.group.WORLD
    dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["tiles", "spp"])
def test_render_distributed_over_nccl_matches_single_gpu(nccl_group, mode):
    import paper_2407_19977_b200 as m
    from paper_2407_19977_b200.distributed import render_distributed
    g = golden_scene("sphere20k")
    st = m.RenderSettings(samples_per_pixel=6, max_depth=5, seed=9)
    ds = m.DeviceScene(g.scene, g.bvh)
    ref = m.render_progressive(ds, st)
    res = render_distributed(ds, st, mode=mode, tile_size=8)
    assert np.array_equal(res.image, ref.image)
    assert np.array_equal(res.invalid_samples, ref.invalid_samples)
