"""Summaries of ncu output for profiles/.

python tools/ncu_summary.py raw REP.ncu-rep [header]   -> selected metrics per launch
python tools/ncu_summary.py launches LAUNCHES.csv [header] -> per-kernel time table

`raw` reads `ncu -i REP --page raw --csv` (the --set full capture);
`launches` reads the --metrics gpu__time_duration.sum --csv launch list.
"""
import collections
import csv
import io
import subprocess
import sys

RAW_METRICS = [
    ("gpu__time_duration.sum", "ms"),
    ("dram__bytes_read.sum", ""),
    ("dram__bytes_write.sum", ""),
    ("lts__t_bytes.sum", ""),
    ("l1tex__t_bytes.sum", ""),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", ""),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "%"),
    ("smsp__inst_executed.sum", "inst"),
    ("l1tex__t_sector_hit_rate.pct", "%"),
    ("lts__t_sector_hit_rate.pct", "%"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "%"),
    ("launch__registers_per_thread", ""),
    ("launch__occupancy_limit_registers", ""),
    ("launch__grid_size", ""),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "%"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "%"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "%"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "%"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "%"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "%"),
]
STALLS = ["long_scoreboard", "wait", "not_selected", "selected", "math_pipe_throttle",
          "short_scoreboard", "branch_resolving", "no_instructions", "lg_throttle",
          "mio_throttle", "barrier", "membar"]


def raw(rep: str, header: str) -> None:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    names, units, data = rows[0], rows[1], rows[2:]
    col = {n: i for i, n in enumerate(names)}
    print(f"# {header}")
    kn = col.get("Kernel Name")
    if kn is not None:
        print(f"{'kernel':58s} {[r[kn][:40] for r in data]}")
    for m, _ in RAW_METRICS:
        if m in col:
            print(f"{m:58s} {[r[col[m]] for r in data]} {units[col[m]]}")
    for s in STALLS:
        m = f"smsp__pcsamp_warps_issue_stalled_{s}"
        if m in col:
            print(f"{'stall_' + s:58s} {[r[col[m]] for r in data]}")


def launches(path: str, header: str) -> None:
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if d.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(d["Metric Value"].replace(",", ""))
        scale = {"ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0}.get(
            d.get("Metric Unit", "ns"), 1e-6)
        name = d["Kernel Name"][:52]
        n, t = tot.get(name, (0, 0.0))
        tot[name] = (n + 1, t + v * scale)
    total = sum(t for _, t in tot.values())
    print(f"# {header}")
    for name, (n, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
        print(f"{name:52s} {n:6d} {t:10.2f} ms {100 * t / total:6.2f}%")
    print(f"{'total':52s} {sum(n for n, _ in tot.values()):6d} {total:10.2f} ms")


if __name__ == "__main__":
    kind, path = sys.argv[1], sys.argv[2]
    head = sys.argv[3] if len(sys.argv) > 3 else path
    {"raw": raw, "launches": launches}[kind](path, head)
