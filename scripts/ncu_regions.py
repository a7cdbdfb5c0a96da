"""Instruction / stall-sample share per kernel region (rqa_unit.cuh line
ranges found by marker comments) of an ncu --import-source report."""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
src = open("paper_2402_16853_b200/csrc/rqa_unit.cuh").read().splitlines()
marks = [("chunk_rows", "auto chunk_rows"), ("diag_pass", "auto diag_pass"),
         ("phase1 (predicate + candidates)", "if constexpr (kPre) {"),
         ("phase2", "// ---- phase 2"), ("generic eval", "uint32_t wprev[R];"),
         ("row phase", "// ---- row phase"), ("column phase", "// ---- column phase"),
         ("diag end", "// ---- diagonal pieces"), ("tail", "// ---- row pieces")]
starts = []
for name, m in marks:
    for i, line in enumerate(src):
        if m.strip() in line:
            starts.append((i + 1, name))
            break
starts.sort()
def region(ln):
    r = "setup"
    for s, name in starts:
        if ln >= s:
            r = name
    return r
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname = "?"
agg = collections.Counter()
smp = collections.Counter()
for rec in csv.reader(out.splitlines()):
    if not rec:
        continue
    if rec[0] == "File Path":
        fname = rec[1].split("/")[-1]
        continue
    if rec[0] in ("Line No", "Function Name") or len(rec) < 8 or rec[2] != "-":
        continue
    try:
        inst, s, ln = int(rec[7] or 0), int(rec[4] or 0), int(rec[0])
    except ValueError:
        continue
    key = region(ln) if fname == "rqa_unit.cuh" else fname
    agg[key] += inst
    smp[key] += s
ti, ts = sum(agg.values()), sum(smp.values())
for k, v in agg.most_common():
    print(f"{100 * v / ti:5.1f}% inst {100 * smp[k] / ts:5.1f}% samples  {k}")
