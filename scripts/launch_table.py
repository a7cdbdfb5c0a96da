"""Per-kernel launch count and mean time of an ncu --metrics gpu__time_duration.sum CSV."""
import collections
import csv
import sys

agg = collections.defaultdict(list)
for r in csv.DictReader(line for line in open(sys.argv[1]) if not line.startswith("==")):
    if r.get("Metric Name") == "gpu__time_duration.sum":
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        agg[r["Kernel Name"][:70]].append(v * {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0,
                                                "msecond": 1.0}.get(unit, 1.0))
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):4d} x {sum(v) / len(v):10.3f} ms  {k}")
