"""ncu figures of k_trace for bench.py's roofline (profiles/trace_ncu.json).

On the GPU box (one GPU, after the same pass ran clean without ncu):
  python tools/trace_ncu.py capture [--workload pushbutton] [--spp 32]
      -> gpurun_out/trace_ncu_<workload>.csv / .log: the 8 k_trace launches
         (depths 0..7) of one whole-frame batch on one lane, with the
         per-level byte counters and the unit utilisations below
Here:
  python tools/trace_ncu.py summarize gpurun_out/trace_ncu_<workload>.csv
      -> profiles/trace_ncu.json[<workload>]: bytes per ray per memory level
         (sums over the launches / the batch's rays) and duration-weighted
         utilisations, tagged with the kernel sources' hash (bench.py only
         uses figures whose hash matches the sources it times)
"""
import argparse
import ast
import csv
import json
import re
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

SUMS = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "gpu__time_duration.sum", "smsp__inst_executed.sum"]
PCTS = {
    "l1_wavefront_pct": "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "fma_pipe_pct": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "alu_pipe_pct": "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "lsu_pipe_pct": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "l2_throughput_pct": "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "simt_threads": "smsp__thread_inst_executed_per_inst_executed.ratio",
}
UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9,
         "us": 1e-6, "ms": 1e-3,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def capture(a):
    out = ROOT / "gpurun_out"
    out.mkdir(exist_ok=True)
    csv_path = out / f"trace_ncu_{a.workload}.csv"
    log_path = out / f"trace_ncu_{a.workload}.log"
    cmd = ["ncu", "--metrics", ",".join(SUMS + list(PCTS.values())), "--clock-control", "none",
           "-k", "regex:k_trace", "-c", "8", "--csv", "--log-file", str(csv_path),
           sys.executable, str(ROOT / "tools" / "profile_pass.py"), "--workload", a.workload,
           "--spp", str(a.spp)]
    with open(log_path, "w") as log:
        subprocess.run(cmd, stdout=log, stderr=subprocess.STDOUT, check=True,
                       env={**__import__("os").environ, "LT_LANES": "1"})


def summarize(a):
    from bench import trace_source_sha
    per = {}
    hdr = None
    for r in csv.reader(open(a.csv)):
        if "Metric Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", "")) * UNITS.get(d["Metric Unit"], 1.0)
        per.setdefault(d["ID"], {})[d["Metric Name"]] = v
    launches = list(per.values())
    log = Path(a.csv).with_suffix(".log").read_text()
    rays = ast.literal_eval(re.search(r"stats (\{.*\})", log).group(1))["rays"]
    tot = {m: sum(x.get(m, 0.0) for x in launches) for m in SUMS}
    dur = tot["gpu__time_duration.sum"]
    entry = {
        "dram_bytes_per_ray": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / rays,
        "l2_bytes_per_ray": tot["lts__t_bytes.sum"] / rays,
        "l1_bytes_per_ray": tot["l1tex__t_bytes.sum"] / rays,
        "instructions_per_ray": tot["smsp__inst_executed.sum"] / rays,
        "rays": rays, "launches": len(launches),
        "ncu_serialized_ms": dur * 1e3,
        "source_sha": trace_source_sha(),
        "source": f"profiles/r02_trace_ncu_{a.workload}.csv: ncu of the {len(launches)} k_trace launches of one whole-frame "
                  f"batch ({rays} rays, LT_LANES=1, tools/trace_ncu.py)",
    }
    for k, m in PCTS.items():
        entry[k] = sum(x.get(m, 0.0) * x["gpu__time_duration.sum"] for x in launches) / dur
    f = ROOT / "profiles" / "trace_ncu.json"
    data = json.loads(f.read_text()) if f.exists() else {}
    data[a.workload] = entry
    f.write_text(json.dumps(data, indent=1) + "\n")
    print(json.dumps(entry, indent=1))


if __name__ == "__main__":
    p = argparse.ArgumentParser()
    sub = p.add_subparsers(dest="cmd", required=True)
    c = sub.add_parser("capture")
    c.add_argument("--workload", default="pushbutton")
    c.add_argument("--spp", type=int, default=32)
    s = sub.add_parser("summarize")
    s.add_argument("csv")
    s.add_argument("--workload", default="pushbutton")
    a = p.parse_args()
    {"capture": capture, "summarize": summarize}[a.cmd](a)
