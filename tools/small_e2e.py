"""Per-call overheads of render_progressive on the tiny C1 workload."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_19977_b200 import RenderSettings, build_bvh, render_progressive  # noqa: E402
from workloads import scene_by_name  # noqa: E402

scene = scene_by_name("cornell_c1")
bvh = build_bvh(scene.triangles)
st = RenderSettings(samples_per_pixel=4, max_depth=4, rr_start_depth=3, seed=0)
for rep in range(6):
    t0 = time.perf_counter()
    res = render_progressive(scene, st, bvh=bvh)
    print(f"rep {rep}: {1e3 * (time.perf_counter() - t0):7.3f} ms  "
          + ", ".join(f"{k} {v:.3f}" for k, v in res.timings.items()), flush=True)
