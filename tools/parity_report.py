"""Fold the parity lines the -m gpu tests append (gpurun_out/parity_r02.jsonl)
into the committed profiles/parity_r02.json.

python tools/parity_report.py [gpurun_out/parity_r02.jsonl]

Keeps the latest line per (test, scene, sample) key; `headline` summarizes
the C4 figures the bench line quotes.
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def main():
    src = Path(sys.argv[1] if len(sys.argv) > 1 else ROOT / "gpurun_out" / "parity_r02.jsonl")
    entries = {}
    for line in src.read_text().splitlines():
        if not line.strip():
            continue
        d = json.loads(line)
        key = "/".join(str(d[k]) for k in ("test", "scene", "sample") if k in d)
        entries[key] = d
    head = {}
    for key, d in entries.items():
        if d["test"] == "headline_per_sample":
            head[d["scene"]] = {
                "rows": d["all"]["rows"],
                "frac_le_1e-4_all": d["all"]["frac_le_0.0001"],
                "frac_le_1e-4_excluding_near_mirror": d["excluding_near_mirror"]["frac_le_0.0001"],
                "frac_le_1e-3_all": d["all"]["frac_le_0.001"],
                "rows_gt_1e-3": d["all"]["count_gt_0.001"],
                "near_mirror_rows": d["near_mirror_rows"],
                "near_mirror_frac_le_1e-4": d["near_mirror_primary"]["frac_le_0.0001"],
            }
        if d["test"] == "headline_primary_ids":
            h = head.setdefault("primary_ids_pushbutton_ref", {"rays": 0, "id_mismatches": 0})
            h["rays"] += d["rays"]
            h["id_mismatches"] += d["id_mismatches"]
            h["ppm"] = 1e6 * h["id_mismatches"] / h["rays"]
    out = {"source": f"{src.name}: lines appended by tests/test_gpu_headline_parity.py and "
                     "tests/test_gpu_parity.py on the B200 (python -m pytest tests -m gpu)",
           "tolerance": "per (pixel, sample) row: |gpu - oracle| <= rel * max(1, |oracle|) on "
                        "all three channels; fractions per rel in each entry",
           "headline": head, "entries": entries}
    dst = ROOT / "profiles" / "parity_r02.json"
    dst.write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(head, indent=1))


if __name__ == "__main__":
    main()
