"""Per-CUDA-source-line instruction counts and stall samples of an ncu report
(ncu --set full --import-source on).  usage: ncu_lines.py REPORT [TOP]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = []
fname = "?"
hdr = None
for rec in csv.reader(out.splitlines()):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] == "Line No":
        hdr = rec
        continue
    if hdr is None or rec[0] in ("Function Name",) or len(rec) < 8:
        continue
    if rec[2] != "-":
        continue
    try:
        samples = int(rec[4] or 0)
        inst = int(rec[7] or 0)
    except ValueError:
        continue
    rows.append((inst, samples, fname, rec[0], rec[1].strip()[:90]))
ti = sum(r[0] for r in rows) or 1
ts = sum(r[1] for r in rows) or 1
print(f"total warp instructions {ti:.4g}, stall samples {ts}")
for inst, samp, f, ln, src in sorted(rows, key=lambda r: -r[1])[:top]:
    print(f"{100 * samp / ts:5.1f}% smp {100 * inst / ti:5.1f}% inst  {f}:{ln}  {src}")
