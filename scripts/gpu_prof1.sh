#!/bin/bash
# ncu --set full with source of the hot kernel on one workload (prefix).
TAG=${1:-p}; WL=${2:-C3}; PRE=${3:-262146}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"unit_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_${WL}_${TAG} python scripts/profile_once.py ${WL} 2 ${PRE} > gpurun_out/prof_${WL}_${TAG}.log 2>&1
tail -1 gpurun_out/prof_${WL}_${TAG}.log
