"""Material-class divergence of the shade warps (LT_FLAG_COUNT): how many
warps see more than one material class among their active lanes.  Evidence
for / against sorting shade work by material (BASELINE north star)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_2407_19977_b200 import RenderSettings, build_bvh  # noqa: E402
from paper_2407_19977_b200._lib import LT_FLAG_COUNT  # noqa: E402
from paper_2407_19977_b200.device import DeviceScene  # noqa: E402
from paper_2407_19977_b200.integrator import Accumulator, render_pass_device  # noqa: E402
from workloads import scene_by_name  # noqa: E402

for name in sys.argv[1:] or ["pushbutton", "cornell_c2x", "sphere70k"]:
    scene = scene_by_name(name, width=1920, height=1080) if name in ("pushbutton", "sphere70k") \
        else scene_by_name(name)
    ds = DeviceScene(scene, build_bvh(scene.triangles))
    cam = scene.camera
    acc = Accumulator(cam.width, cam.height, 0)
    st = RenderSettings(samples_per_pixel=4, max_depth=8, rr_start_depth=3, seed=0)
    for octant in (1,):
        render_pass_device(ds, cam, st, acc, 0, 4, flags=LT_FLAG_COUNT)
        s = ds.stats()
        w = max(1, s["shade_warps"])
        print(f"{name}: {len(scene.triangles)} tris, {len(scene.materials)} materials: "
              f"{s['shade_warps']} shade warps, {100 * s['shade_mixed_warps'] / w:.1f} % span "
              f">1 material class, {s['shade_warp_classes'] / w:.3f} classes per warp",
              flush=True)
