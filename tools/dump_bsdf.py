"""Dump the device BSDF sample outputs on the golden cases (GPU box)."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from paper_2407_19977_b200.bsdf import eval_pdf_batch, sample_batch  # noqa: E402

z = np.load(ROOT / "tests" / "golden" / "material.npz")
ext = [0.0, 0.0, 1.5, 1.0, 1.0, 1.0, 0.0, 1.0, 1.0, 1.0]
params = np.hstack([z["params"], np.tile(ext, (len(z["params"]), 1))])
rows = z["rows"]
ok, wi, w = sample_batch(params, rows[:, 0:3], rows[:, 3:6], rows[:, 6:9])
f, pdf = eval_pdf_batch(params, rows[:, 0:3], rows[:, 18:21], rows[:, 3:6])
(ROOT / "gpurun_out").mkdir(exist_ok=True)
np.savez(ROOT / "gpurun_out" / "bsdf_dump.npz", ok=ok, wi=wi, w=w, f=f, pdf=pdf)
print("dumped", ok.shape)
