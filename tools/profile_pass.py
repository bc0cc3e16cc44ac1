"""One render pass of the bench workload for profiler captures (ncu -k ...).

python tools/profile_pass.py [--spp 16] [--warm 1]: builds C4, runs `warm`
untimed passes, then one pass; prints its wall time.  Kernel-level numbers
come from the profiler, never from this script's clock.
"""
import argparse
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main():
    p = argparse.ArgumentParser()
    p.add_argument("--workload", default="pushbutton")
    p.add_argument("--spp", type=int, default=16)
    p.add_argument("--warm", type=int, default=0)
    p.add_argument("--depth", type=int, default=8)
    a = p.parse_args()
    import torch
    from paper_2407_19977_b200 import RenderSettings, build_bvh
    from paper_2407_19977_b200.device import DeviceScene
    from paper_2407_19977_b200.integrator import Accumulator, render_pass_device
    from workloads import scene_by_name
    scene = scene_by_name(a.workload, width=1920, height=1080)
    bvh = build_bvh(scene.triangles)
    ds = DeviceScene(scene, bvh)
    cam = scene.camera
    acc = Accumulator(cam.width, cam.height, 0)
    st = RenderSettings(samples_per_pixel=a.spp, max_depth=a.depth, rr_start_depth=3, seed=0)
    for _ in range(a.warm + 1):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        render_pass_device(ds, cam, st, acc, 0, a.spp)
        torch.cuda.synchronize()
    print(f"pass {a.spp} spp: {1e3 * (time.perf_counter() - t0):.1f} ms; stats {ds.stats()}")


if __name__ == "__main__":
    main()
