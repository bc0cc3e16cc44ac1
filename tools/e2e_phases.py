"""Phase timing of one end-to-end render_progressive call (GPU box)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2407_19977_b200 import RenderSettings, build_bvh  # noqa: E402
from paper_2407_19977_b200.device import DeviceScene  # noqa: E402
from paper_2407_19977_b200.integrator import Accumulator, render_pass_device  # noqa: E402
from paper_2407_19977_b200.procgen import scene_by_name  # noqa: E402

sc = scene_by_name("pushbutton")
bvh = build_bvh(sc.triangles)
st = RenderSettings(samples_per_pixel=256, max_depth=8, rr_start_depth=3, seed=0)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ds = DeviceScene(sc, bvh)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    acc = Accumulator(1920, 1080, 0)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    render_pass_device(ds, sc.camera, st, acc, 0, 256)
    t3 = time.perf_counter()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    img = acc.mean().cpu().numpy()
    inv = acc.invalid.cpu().numpy()
    t5 = time.perf_counter()
    del ds
    torch.cuda.synchronize()
    t6 = time.perf_counter()
    print(f"iter {it}: scene {1e3*(t1-t0):.1f} ms, acc alloc {1e3*(t2-t1):.1f}, enqueue "
          f"{1e3*(t3-t2):.1f}, render wait {1e3*(t4-t3):.1f}, image D2H {1e3*(t5-t4):.1f}, "
          f"destroy {1e3*(t6-t5):.1f}", flush=True)
