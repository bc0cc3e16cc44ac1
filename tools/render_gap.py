"""Where does a single render_progressive frame lose time against the
device-timed bench step?  (GPU box; prints wall / event times.)"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2407_19977_b200 import RenderSettings, build_bvh, render_progressive  # noqa: E402
from paper_2407_19977_b200.device import DeviceScene  # noqa: E402
from paper_2407_19977_b200.integrator import Accumulator, render_pass_device  # noqa: E402
from workloads import scene_by_name  # noqa: E402

scene = scene_by_name("pushbutton")
bvh = build_bvh(scene.triangles)
st = RenderSettings(samples_per_pixel=256, max_depth=8, rr_start_depth=3, seed=0)
ds = DeviceScene(scene, bvh)
cam = scene.camera
acc = Accumulator(cam.width, cam.height, 0)
stream = torch.cuda.current_stream()


def timed(fn, label, reps=4):
    for r in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(stream)
        fn()
        e1.record(stream)
        torch.cuda.synchronize()
        print(f"{label:42s} rep {r}: wall {1e3 * (time.perf_counter() - t0):7.1f} ms, "
              f"events {e0.elapsed_time(e1):7.1f} ms", flush=True)


def one_pass():
    acc.sum.zero_()
    acc.valid.zero_()
    acc.invalid.zero_()
    render_pass_device(ds, cam, st, acc, 0, 256, stream=stream)


timed(one_pass, "render_pass_device, sync each")
timed(lambda: render_progressive(ds, st), "render_progressive(resident scene)")


def four():
    for _ in range(4):
        one_pass()


timed(four, "4 x render_pass_device back to back", reps=2)
timed(lambda: render_progressive(scene, st, bvh=bvh), "render_progressive(host scene)")

# first renders on freshly created scenes (creation excluded from the timing)
for rep in range(3):
    fresh = DeviceScene(scene, bvh)
    torch.cuda.synchronize()
    timed(lambda: render_progressive(fresh, st), f"fresh scene {rep}: render_progressive", reps=2)
    fresh.close()
