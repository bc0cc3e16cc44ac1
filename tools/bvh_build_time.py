"""Time build_bvh on the GPU vs the host restatement (GPU box)."""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2407_19977_b200 import build_bvh  # noqa: E402
from workloads import scene_by_name  # noqa: E402

for name in sys.argv[1:] or ["pushbutton", "sphere70k"]:
    tris = scene_by_name(name, width=64, height=36).triangles
    for dev in [0, 0, 0, None]:
        t0 = time.perf_counter()
        b = build_bvh(tris, device=dev)
        print(f"{name} {len(tris)} tris device={dev}: {1e3 * (time.perf_counter() - t0):.1f} ms "
              f"({b.stats.node_count} nodes)", flush=True)
