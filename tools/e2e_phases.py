"""Phase timing of end-to-end render_progressive calls (GPU box): the scene's
plain numpy arrays (pageable, as a luxtrace caller holds them), or with
--pinned page-locked copies."""
import gc
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_19977_b200 import RenderSettings, build_bvh, render_progressive  # noqa: E402
from workloads import scene_by_name  # noqa: E402


def pin(obj, names, keep):
    for nm in names:
        a = np.ascontiguousarray(getattr(obj, nm))
        t = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, pin_memory=True)
        t.numpy()[...] = a
        keep.append(t)
        setattr(obj, nm, t.numpy())


sc = scene_by_name("pushbutton")
bvh = build_bvh(sc.triangles)
keep = []
if "--pinned" in sys.argv:
    pin(sc.triangles, ["v0", "v1", "v2", "n0", "n1", "n2", "material_index"], keep)
    pin(bvh, ["bounds_min", "bounds_max", "left_child", "right_child", "first_triangle",
              "triangle_count", "triangle_order"], keep)
    if sc.environment.texels is not None:
        pin(sc.environment, ["texels"], keep)
st = RenderSettings(samples_per_pixel=256, max_depth=8, rr_start_depth=3, seed=0)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = render_progressive(sc, st, bvh=bvh)
    t1 = time.perf_counter()
    print({k: round(v, 1) for k, v in res.timings.items()}, flush=True)
    del res
    gc.collect()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"iter {it}: call {1e3*(t1-t0):.1f} ms, release {1e3*(t2-t1):.1f} ms", flush=True)
    sys.stdout.flush()
