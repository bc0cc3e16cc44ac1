"""Benchmark-harness fixtures (luxtrace bench.py) produced by the reference.

Run in the build container (the reference is importable there):
    NUMBA_CACHE_DIR=/tmp/numba PYTHONPATH=/root/reference/pkg/src \
        python tests/golden/make_harness_golden.py
Writes tests/golden/harness_expected.json: summarize_runs / format_ms
values, a formatted report table and JSON document, and the auto-framing
camera and scene summary load_benchmark_scene gives the ingest fixtures.
"""
import json
from pathlib import Path

import numpy as np

from luxtrace import bench  # noqa: E402  (the reference)

HERE = Path(__file__).resolve().parent
runs = [327.125, 328.5, 326.75, 329.0, 327.25]
mean, sd = bench.summarize_runs(runs)
rep = bench.BenchmarkReport(machine="test-machine", settings={"runs": 5, "spp": 100})
rep.rows.append(bench.BenchRow(1068735, bench.PHASE_BUILD, mean, sd, 5))
rep.rows.append(bench.BenchRow(10687, bench.PHASE_TRACE, 790.83, 4.18, 30))
out = {"runs": runs, "mean": mean, "stddev": sd, "format": bench.format_ms(mean, sd),
       "table": rep.format_table(), "json": rep.to_json_document(), "scenes": {}}
for name in ("ico.glb", "hier.glb"):
    sc = bench.load_benchmark_scene(HERE / "ingest" / name, 320, 200)
    cam = sc.camera
    out["scenes"][name] = {
        "position": [float(x) for x in cam.position], "look_at": [float(x) for x in cam.look_at],
        "fov": cam.vertical_fov_deg, "width": cam.width, "height": cam.height,
        "env_kind": sc.environment.kind, "zenith": [float(x) for x in sc.environment.zenith],
        "horizon": [float(x) for x in sc.environment.horizon],
        "n_triangles": len(sc.triangles), "dropped": sc.degenerate_dropped,
        "v_sum": float(np.sum(sc.triangles.v0) + np.sum(sc.triangles.v1) + np.sum(sc.triangles.v2))}
(HERE / "harness_expected.json").write_text(json.dumps(out, indent=1) + "\n")
print("wrote harness_expected.json")
