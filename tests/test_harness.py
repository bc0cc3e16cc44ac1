"""The benchmark-harness API (reference bench.py) against fixtures the
reference produced (tests/golden/make_harness_golden.py): statistics, the
report's text and JSON forms, the auto-framing camera and the benchmark
scene loader.  The GPU test runs a tiny benchmark end to end."""
from __future__ import annotations

import json

import numpy as np
import pytest

from conftest import GOLDEN

Z = json.loads((GOLDEN / "harness_expected.json").read_text())


def test_statistics_and_formatting():
    import paper_2407_19977_b200 as lb
    mean, sd = lb.summarize_runs(Z["runs"])
    assert mean == Z["mean"] and sd == Z["stddev"]
    assert lb.format_ms(mean, sd) == Z["format"]
    with pytest.raises(ValueError, match="at least 2 runs"):
        lb.summarize_runs([1.0])


def test_report_table_and_json():
    import paper_2407_19977_b200 as lb
    from paper_2407_19977_b200.harness import PHASE_BUILD, PHASE_TRACE
    rep = lb.BenchmarkReport(machine="test-machine", settings={"runs": 5, "spp": 100})
    rep.rows.append(lb.BenchRow(1068735, PHASE_BUILD, Z["mean"], Z["stddev"], 5))
    rep.rows.append(lb.BenchRow(10687, PHASE_TRACE, 790.83, 4.18, 30))
    assert rep.format_table() == Z["table"]
    assert rep.to_json_document() == Z["json"]


@pytest.mark.parametrize("name", ["ico.glb", "hier.glb"])
def test_benchmark_scene_and_camera(name):
    import paper_2407_19977_b200 as lb
    sc = lb.load_benchmark_scene(GOLDEN / "ingest" / name, 320, 200)
    want = Z["scenes"][name]
    cam = sc.camera
    assert list(map(float, cam.position)) == want["position"]
    assert list(map(float, cam.look_at)) == want["look_at"]
    assert (cam.vertical_fov_deg, cam.width, cam.height) == (want["fov"], want["width"],
                                                              want["height"])
    env = sc.environment
    assert env.kind == want["env_kind"]
    assert list(map(float, env.zenith)) == want["zenith"]
    assert list(map(float, env.horizon)) == want["horizon"]
    assert len(sc.triangles) == want["n_triangles"] and sc.degenerate_dropped == want["dropped"]
    t = sc.triangles
    assert float(np.sum(t.v0) + np.sum(t.v1) + np.sum(t.v2)) == want["v_sum"]


def test_run_benchmark_argument_errors():
    import paper_2407_19977_b200 as lb
    with pytest.raises(ValueError, match="at least 2 runs"):
        lb.run_benchmark([], runs=1)
    with pytest.raises(ValueError, match="warmup"):
        lb.run_benchmark([], warmup=-1)


@pytest.mark.gpu
def test_run_benchmark_on_the_gpu(tmp_path):
    """Both phases of a tiny benchmark run through this package's GPU BVH
    build and renderer; the report has one row per (scene, phase)."""
    import paper_2407_19977_b200 as lb
    msgs = []
    paths = [GOLDEN / "ingest" / "ico.glb", GOLDEN / "ingest" / "hier.glb"]
    rep = lb.run_benchmark(paths, runs=3, spp=4, warmup=1, width=64, height=48,
                           progress=msgs.append)
    assert [r.phase for r in rep.rows] == ["bvh_build", "trace"] * 2
    assert all(r.run_count == 3 and r.mean_ms > 0.0 for r in rep.rows)
    assert len(msgs) == 4 and "over 3 runs" in msgs[0]
    rep.write_json(tmp_path / "r.json")
    assert json.loads((tmp_path / "r.json").read_text())["settings"]["spp"] == 4
    assert "bvh_build" in rep.format_table()
