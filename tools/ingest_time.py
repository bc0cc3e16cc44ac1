"""GLB -> resident scene: host ingest vs device ingest.

  host    load_scene (numpy float64 flatten, the reference's path) then
          DeviceScene(scene) (upload of the float64 soup + device BVH build)
  device  load_device_scene: JSON + node walk on the host, raw GLB bytes up,
          flatten + BVH build on the device (lt_scene_create_gltf)
  gpu_sd  load_scene_gpu: the device flatten with the soup copied back (a
          SceneDescription, bit-identical to load_scene's)

Wall-clock per call (the caller's view), median of --reps after one warm-up,
on the C4 pushbutton written as a GLB with explicit / generated normals.
python tools/ingest_time.py [--reps 5]
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    a = ap.parse_args()
    import torch

    import workloads
    import paper_2407_19977_b200 as lb
    from paper_2407_19977_b200.ingest import load_device_scene, load_scene, load_scene_gpu
    sc = workloads.pushbutton()
    tmp = Path(tempfile.mkdtemp())
    for normals in (True, False):
        glb, cfg = tmp / f"pb{int(normals)}.glb", tmp / f"pb{int(normals)}.json"
        workloads.write_gltf(sc, glb, cfg, normals=normals)

        def host():
            sd = load_scene(glb, cfg)
            ds = lb.DeviceScene(sd)
            torch.cuda.synchronize()
            return ds

        def device():
            ds = load_device_scene(glb, cfg)
            torch.cuda.synchronize()
            return ds

        def gpu_sd():
            return load_scene_gpu(glb, cfg)

        out = {"workload": "pushbutton GLB", "normals": "explicit" if normals else "generated",
               "glb_bytes": glb.stat().st_size}
        for name, fn in (("host", host), ("device", device), ("gpu_sd", gpu_sd)):
            r = fn()
            if name != "gpu_sd":
                out["n_triangles"] = r.n_triangles
                r.close()
            ts = []
            for _ in range(a.reps):
                t0 = time.perf_counter()
                r = fn()
                ts.append((time.perf_counter() - t0) * 1e3)
                if name != "gpu_sd":
                    r.close()
            out[f"{name}_ms"] = round(statistics.median(ts), 1)
        # the host half of the device path alone
        from paper_2407_19977_b200.ingest import (gltf_device_desc, load_gltf_located,
                                                  load_render_config)
        ts = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            gltf_device_desc(load_gltf_located(glb), load_render_config(cfg).materials)
            ts.append((time.perf_counter() - t0) * 1e3)
        out["device_host_part_ms"] = round(statistics.median(ts), 1)
        out["speedup_resident"] = round(out["host_ms"] / out["device_ms"], 1)
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
