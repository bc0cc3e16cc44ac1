"""Per-ray memory traffic of k_trace from an ncu metrics CSV.

The capture (one GPU, after the same command ran clean without ncu):
  LT_LANES=1 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,\
l1tex__t_bytes.sum --clock-control none -k regex:k_trace -c 8 --csv --log-file T.csv \
      python tools/profile_pass.py --spp 32 > T.log
(one 66 M-path batch = the 8 trace launches of depths 0..7).

python tools/trace_traffic.py T.csv T.log SOURCE_NOTE -> updates profiles/trace_traffic.json
"""
import ast
import csv
import json
import re
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
UNITS = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def main():
    csv_path, log_path, note = sys.argv[1], sys.argv[2], sys.argv[3]
    tot = {}
    hdr = None
    for r in csv.reader(open(csv_path)):
        if "Metric Name" in r:
            hdr = r
            continue
        if hdr is None or len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        v = float(d["Metric Value"].replace(",", "")) * UNITS.get(d["Metric Unit"], 1.0)
        tot[d["Metric Name"]] = tot.get(d["Metric Name"], 0.0) + v
    m = re.search(r"stats (\{.*\})", Path(log_path).read_text())
    rays = ast.literal_eval(m.group(1))["rays"]
    out_path = ROOT / "profiles" / "trace_traffic.json"
    data = json.loads(out_path.read_text()) if out_path.exists() else {}
    data["pushbutton"] = {
        "dram_bytes_per_ray": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / rays,
        "l2_bytes_per_ray": tot["lts__t_bytes.sum"] / rays,
        "l1_bytes_per_ray": tot["l1tex__t_bytes.sum"] / rays,
        "rays": rays,
        "source": note,
    }
    out_path.write_text(json.dumps(data, indent=1) + "\n")
    print(json.dumps(data["pushbutton"], indent=1))


if __name__ == "__main__":
    main()
