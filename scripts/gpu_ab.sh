#!/bin/bash
# A/B: parity subset with each variant, then interleaved timings.
# VARIANTS="base x" WLS="C3 P C4" ROUNDS=2 bash scripts/gpu_ab.sh
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
for v in ${VARIANTS}; do
  echo -n "$v parity: "; RQA_LIB_PATH=$PWD/abtest/$v/librqa_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -m gpu -q -x -p no:cacheprovider 2>&1 | grep -E "passed|failed" | tail -1
done
bash scripts/ab_time.sh
