#!/bin/bash
# RQA_SKIP phase ablation (profiling only: results are wrong when a phase is skipped)
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for S in 0 1 2 4 7; do
  echo -n "skip=$S "; RQA_SKIP=$S timeout 300 python scripts/time_configs.py ${WLS:-C3} 2>&1 | tail -1
done
