#!/bin/bash
# compute-sanitizer evidence: memcheck, racecheck, synccheck, initcheck over scripts/sanitize_cases.py
# (kept for reference: the GPU pool has since closed compute-sanitizer; use gpu_checked.sh)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
export RQA_PREFILTER=${RQA_PREFILTER:-1}
# empty the shared bins every 2 iterations: exercises the mid-unit flush path
export RQA_FLUSH_EVERY=${RQA_FLUSH_EVERY:-2}
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize_cases.py ${N:-1200} > gpurun_out/sanitize_${tool}.txt 2>&1
  echo "$tool rc=$?"; tail -4 gpurun_out/sanitize_${tool}.txt
done
