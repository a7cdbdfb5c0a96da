"""Summarise an ncu report: key metrics, opcode mix, instruction share by region."""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
d = dict(zip(raw[0], raw[2]))
keys = ["gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__inst_executed.avg.per_cycle_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_fp64.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__grid_size", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "smsp__thread_inst_executed_per_inst_executed.ratio"]
for k in keys:
    if k in d:
        print(f"{k:70s} {d[k]}")
for k in sorted(d):
    if "average_warps_issue_stalled" in k and "per_issue_active" in k:
        try:
            v = float(d[k])
        except ValueError:
            continue
        if v > 0.05:
            print(f"{k:70s} {v:.2f}")
txt = ncu("--page", "raw", "--print-metric-instances", "details", "--metrics", "sass__inst_executed_per_opcode")
body = txt[txt.find("(") + 1: txt.rfind(")")]
ops = [x.strip() for x in body.replace("\n", " ").split(";")]
pairs = []
for o in ops:
    if ":" in o:
        name, val = o.rsplit(":", 1)
        try:
            pairs.append((name.strip(), int(val.strip())))
        except ValueError:
            pass
tot = sum(v for _, v in pairs) or 1
print("opcode mix:", ", ".join(f"{n} {v / tot:.1%}" for n, v in sorted(pairs, key=lambda x: -x[1])[:22]))
