"""Shared test fixtures.

Markers: `gpu` tests need a CUDA device (run on the B200 via gpurun); the
rest run on CPU.  Golden fixtures (tests/golden/*.npz) were produced by the
reference itself (tests/golden/make_golden.py).
"""
from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

SCENES = ["floor", "shell", "glossy", "sphere2k", "dup", "cornell_c1", "cornell_c2", "sphere20k"]


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def gpu_available() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class GoldenScene:
    """One reference fixture: inputs as package objects + reference outputs."""

    def __init__(self, name: str):
        from paper_2407_19977_b200 import (Bvh, BuildStats, CameraConfig, EnvironmentConfig,
                                           OpenPbrParams, RenderSettings, SceneDescription,
                                           TriangleBuffer)
        z = np.load(GOLDEN / f"scene_{name}.npz")
        self.name = name
        self.z = z
        self.triangles = TriangleBuffer(z["v0"], z["v1"], z["v2"], z["n0"], z["n1"], z["n2"],
                                        z["material_index"])
        k = z["mat_base_weight"].shape[0]
        self.materials = [OpenPbrParams(
            base_weight=float(z["mat_base_weight"][i]), base_color=tuple(z["mat_base_color"][i]),
            base_metalness=float(z["mat_base_metalness"][i]),
            specular_weight=float(z["mat_specular_weight"][i]),
            specular_color=tuple(z["mat_specular_color"][i]),
            specular_roughness=float(z["mat_specular_roughness"][i]),
            specular_ior=float(z["mat_specular_ior"][i]),
            emission_luminance=float(z["mat_emission_luminance"][i]),
            emission_color=tuple(z["mat_emission_color"][i])) for i in range(k)]
        self.camera = CameraConfig(position=z["cam_position"], look_at=z["cam_look_at"],
                                   up=z["cam_up"], vertical_fov_deg=float(z["cam_fov"]),
                                   width=int(z["width"]), height=int(z["height"]))
        kind = str(z["env_kind"])
        self.environment = (EnvironmentConfig.uniform(z["env_radiance"]) if kind == "uniform"
                            else EnvironmentConfig.gradient(z["env_zenith"], z["env_horizon"]))
        nn = z["bvh_left"].shape[0]
        self.bvh = Bvh(z["bvh_bounds_min"], z["bvh_bounds_max"], z["bvh_left"], z["bvh_right"],
                       z["bvh_first"], z["bvh_count"], z["bvh_order"],
                       BuildStats(nn, int((z["bvh_count"] > 0).sum()), 0, 0.0))
        self.scene = SceneDescription(self.triangles, self.materials, self.camera,
                                      self.environment, 0)
        self.settings = RenderSettings(samples_per_pixel=int(z["spp"]),
                                       max_depth=int(z["max_depth"]),
                                       rr_start_depth=int(z["rr_start"]), seed=int(z["seed"]),
                                       t_min=float(z["t_min"]))

    def __getitem__(self, key):
        return self.z[key]

    def oracle(self):
        from oracle.oracle import OracleScene
        return OracleScene(self.triangles, self.bvh, self.materials, self.environment)


_cache: dict[str, GoldenScene] = {}


def golden_scene(name: str) -> GoldenScene:
    if name not in _cache:
        _cache[name] = GoldenScene(name)
    return _cache[name]


@pytest.fixture(params=SCENES)
def gscene(request):
    return golden_scene(request.param)


@pytest.fixture(scope="session")
def oracle_lib():
    from oracle import oracle
    oracle.build()
    return oracle


# ------------------------------------------------------------------ parity record

PARITY_LOG = ROOT / "gpurun_out" / "parity_r02.jsonl"


def record_parity(test: str, **fields) -> None:
    """Append one parity measurement (agreement fractions, id-mismatch
    counts) to gpurun_out/parity_r02.jsonl; tools/parity_report.py folds the
    lines into the committed profiles/parity_r02.json."""
    import json
    import time
    PARITY_LOG.parent.mkdir(exist_ok=True)
    with open(PARITY_LOG, "a") as f:
        f.write(json.dumps({"test": test, "time": time.strftime("%Y-%m-%dT%H:%M:%S"),
                            **fields}, default=float) + "\n")


def agreement_tiers(got, ref, rels=(1e-5, 1e-4, 1e-3, 1e-2)) -> dict:
    """Fraction of (pixel, sample) rows whose three channels satisfy
    |got - ref| <= rel * max(1, |ref|), per tolerance; rows where both are
    non-finite count as agreeing, exactly one non-finite as disagreeing."""
    got = np.asarray(got).reshape(-1, 3)
    ref = np.asarray(ref).reshape(-1, 3)
    fin_g = np.isfinite(got).all(axis=1)
    fin_r = np.isfinite(ref).all(axis=1)
    both_nan = ~fin_g & ~fin_r
    err = np.abs(np.nan_to_num(got) - np.nan_to_num(ref)) / np.maximum(1.0, np.abs(
        np.nan_to_num(ref)))
    worst = err.max(axis=1)
    out = {"rows": int(got.shape[0]), "nonfinite_mismatch": int(np.sum(fin_g != fin_r))}
    for r in rels:
        ok = (fin_g & fin_r & (worst <= r)) | both_nan
        out[f"frac_le_{r:g}"] = float(ok.mean())
        out[f"count_gt_{r:g}"] = int((~ok).sum())
    return out
