"""render_progressive(scene, settings) without a BVH (the reference's
default call): the scene builds the reference's tree on the device."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_19977_b200 import RenderSettings, build_bvh, render_progressive  # noqa: E402
from workloads import scene_by_name  # noqa: E402

scene = scene_by_name("pushbutton")
st = RenderSettings(samples_per_pixel=256, max_depth=8, rr_start_depth=3, seed=0)
bvh = build_bvh(scene.triangles)
for label, kw in [("with host Bvh", {"bvh": bvh}), ("no BVH (device build)", {})]:
    for rep in range(3):
        t0 = time.perf_counter()
        res = render_progressive(scene, st, **kw)
        print(f"{label:24s} rep {rep}: {1e3 * (time.perf_counter() - t0):7.1f} ms  "
              f"{res.timings}", flush=True)
