"""Update profiles/ncu_traffic.json (read by bench.py) from one ncu --set full
capture of the hot kernel and the ncu launch list of the bench command.

usage: python scripts/update_traffic.py WORKLOAD REPORT.ncu-rep LAUNCHES.csv NOTE
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

wl, rep, launches, note = sys.argv[1], sys.argv[2], sys.argv[3], sys.argv[4]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3}
metrics = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
           "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
           "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(metrics)],
                     capture_output=True, text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]


def get(name):
    i = hdr.index(name)
    return float(vals[i].replace(",", "")) * SCALE.get(units[i], 1.0)


folds = collections.defaultdict(list)
for r in csv.DictReader(line for line in open(launches) if not line.startswith("==")):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        name = r["Kernel Name"]
        for f in ("sym_fold_diag", "unit_fold_hooks", "unit_fold_all", "fix_diag_pieces"):
            if f in name:
                v = float(r["Metric Value"].replace(",", ""))
                folds[f].append(v * (1e-6 if r["Metric Unit"] == "ns" else
                                     1e-3 if r["Metric Unit"] in ("us", "usecond") else 1.0))
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                    "ncu_traffic.json")
data = json.load(open(path)) if os.path.exists(path) else {}
data[wl] = {
    "kernel": vals[hdr.index("Kernel Name")],
    "dram_read_bytes": int(get("dram__bytes_read.sum")),
    "dram_write_bytes": int(get("dram__bytes_write.sum")),
    "gpu_time_ms": get("gpu__time_duration.sum"),
    "warp_instructions": int(get("smsp__inst_executed.sum")),
    "issue_active_pct": get("smsp__issue_active.avg.pct_of_peak_sustained_active"),
    "fp64_pipe_pct": get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    "registers_per_thread": int(get("launch__registers_per_thread")),
    "warps_active_pct": get("sm__warps_active.avg.pct_of_peak_sustained_active"),
    "folds": {f: {"gpu_time_ms": sum(v) / len(v)} for f, v in folds.items() if v},
    "source": {"ncu_report": os.path.basename(rep), "launch_list": os.path.basename(launches)},
    "note": note,
}
json.dump(data, open(path, "w"), indent=1)
print(json.dumps(data[wl], indent=1))
