#!/bin/bash
# ncu --set full of the hot kernel for the given workloads (default C3 C4 P)
TAG=${1:-r02n}; shift; WLS=${*:-C3 C4 P}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for W in $WLS; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"unit_kernel" -s 1 -c 1 \
    -o gpurun_out/${TAG}_ncu_$W python scripts/profile_once.py $W 2 > gpurun_out/${TAG}_ncu_$W.log 2>&1; tail -1 gpurun_out/${TAG}_ncu_$W.log
done
