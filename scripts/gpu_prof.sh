#!/bin/bash
# ncu --set full with source of the hot kernel: C3 prefix and C4 (full).
TAG=${1:-r02p}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"unit_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_C3p_${TAG} python scripts/profile_once.py C3 2 262146 > gpurun_out/prof_C3p_${TAG}.log 2>&1
tail -2 gpurun_out/prof_C3p_${TAG}.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"unit_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_C4_${TAG} python scripts/profile_once.py C4 2 > gpurun_out/prof_C4_${TAG}.log 2>&1
tail -2 gpurun_out/prof_C4_${TAG}.log
