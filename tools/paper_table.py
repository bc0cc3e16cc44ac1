"""The paper's Table 1 benchmark on this package, through the reference's
own harness API (run_benchmark, bench.py:132-187): BVH setup and path-trace
time, 512x512, 100 spp, depth 5, 30 runs after 2 warm-ups, for procedural
scenes with the paper's triangle counts (1,068,735 / 106,873 / 10,687;
PAPER.md:263-287).  The paper's scenes are CAD models; these are
bumpy spheres with the same triangle counts (procgen.bumpy_sphere_glb).

python tools/paper_table.py [--runs 30] [--out profiles/r02_paper_table]
"""
import argparse
import json
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

PAPER = {  # PAPER.md:263-287 (mean ms)
    "bvh_build": {1068735: {"M1 Max": 327.57, "Ryzen 5 5600X": 383.10},
                  106873: {"M1 Max": 45.49, "Ryzen 5 5600X": 41.77},
                  10687: {"M1 Max": 10.53, "Ryzen 5 5600X": 8.43}},
    "trace": {1068735: {"RTX 3080": 1058.73, "M1 Max": 2319.45},
              106873: {"RTX 3080": 790.20, "M1 Max": 1992.11},
              10687: {"RTX 3080": 790.83, "M1 Max": 2031.38}},
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--runs", type=int, default=30)
    ap.add_argument("--out", default=str(ROOT / "gpurun_out" / "paper_table"))
    a = ap.parse_args()
    import paper_2407_19977_b200 as lb
    tmp = Path(tempfile.mkdtemp())
    paths = []
    for n in (1068735, 106873, 10687):
        p = tmp / f"sphere_{n}.glb"
        lb.bumpy_sphere_glb(p, n)
        paths.append(p)
    rep = lb.run_benchmark(paths, runs=a.runs, spp=100, warmup=2, width=512, height=512,
                           max_depth=5, progress=lambda m: print(m, flush=True))
    table = rep.format_table()
    lines = [table, "", "speed-up against the paper's published means (PAPER.md:263-287):"]
    doc = rep.to_json_document()
    doc["paper"] = {ph: {str(k): v for k, v in d.items()} for ph, d in PAPER.items()}
    for r in rep.rows:
        ref = PAPER[r.phase][r.triangle_count]
        lines.append(f"  {r.triangle_count:>9,} {r.phase:<9} {r.mean_ms:9.2f} ms: " + ", ".join(
            f"{hw} {ms:.2f} ms -> {ms / r.mean_ms:.1f}x" for hw, ms in ref.items()))
    text = "\n".join(lines)
    print(text)
    Path(a.out + ".txt").write_text(text + "\n")
    Path(a.out + ".json").write_text(json.dumps(doc, indent=1) + "\n")


if __name__ == "__main__":
    main()
