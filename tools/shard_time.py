"""Per-rank work of an N-GPU tile-sharded frame, timed on one GPU: rank 0's
share (interleaved 16x16 tiles, 1/N of the frame) rendered alone, for the
scaling estimate T(1) / (N * T_rank(N)).  No collective is involved (the
merge is one NCCL reduce of ~33 MB per frame)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2407_19977_b200 import RenderSettings, build_bvh  # noqa: E402
from paper_2407_19977_b200.device import DeviceScene  # noqa: E402
from paper_2407_19977_b200.integrator import Accumulator, render_pass_device  # noqa: E402
from workloads import scene_by_name  # noqa: E402

scene = scene_by_name("pushbutton")
bvh = build_bvh(scene.triangles)
ds = DeviceScene(scene, bvh)
cam = scene.camera
acc = Accumulator(cam.width, cam.height, 0)
st = RenderSettings(samples_per_pixel=256, max_depth=8, rr_start_depth=3, seed=0)
stream = torch.cuda.current_stream()
batch = int(sys.argv[1]) if len(sys.argv) > 1 else 0
base = None
for n in [1, 2, 4, 8]:
    shard = (0, n, 16) if n > 1 else None
    times = []
    for rep in range(4):
        acc.sum.zero_()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        render_pass_device(ds, cam, st, acc, 0, 256, shard=shard, max_batch_paths=batch,
                           stream=stream)
        e1.record(stream)
        torch.cuda.synchronize()
        if rep:
            times.append(e0.elapsed_time(e1))
    t = min(times)
    base = base or t
    print(f"N={n}: rank-0 share {t:8.1f} ms; ideal {base / n:8.1f} ms; "
          f"efficiency {base / (n * t):.3f}  (batch={batch or 'default'}; stats {ds.stats()})",
          flush=True)
