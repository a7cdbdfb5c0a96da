#!/bin/bash
# ncu launch lists (gpu__time_duration) of one analysis per workload: WLS="C3 P C2"
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for W in ${WLS:-C3}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${1:-l}_launches_$W.csv python scripts/profile_once.py $W 2 > /dev/null 2>&1
  echo "== $W"; python scripts/launch_table.py gpurun_out/${1:-l}_launches_$W.csv
done
