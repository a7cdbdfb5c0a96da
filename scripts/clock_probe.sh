#!/bin/bash
# Sample SM clock / power / throttle reasons at 20 Hz while a workload runs.
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-compute-apps=pid,name,used_memory --format=csv
nvidia-smi --query-gpu=clocks.sm,power.draw,clocks_event_reasons.active,temperature.gpu --format=csv,noheader -lms 50 > gpurun_out/clock_probe.csv &
SMI=$!
"$@"
kill $SMI
python - << 'PY'
import collections
rows=[l.strip().split(", ") for l in open("gpurun_out/clock_probe.csv") if l.strip()]
c=collections.Counter((r[0], r[2]) for r in rows)
print(len(rows), "samples"); [print(k, v) for k, v in c.most_common(12)]
PY
