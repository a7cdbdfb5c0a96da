#!/bin/bash
# Parity subset for each abtest/ variant: VARIANTS="a b" bash scripts/gpu_variants_parity.sh
cd "$GRAFT_REPO_ROOT"
for v in ${VARIANTS}; do
  echo -n "$v: "; RQA_LIB_PATH=$PWD/abtest/$v/librqa_b200.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -m gpu -q -p no:cacheprovider 2>&1 | grep -E "passed|failed|RQA_DCHECK" | tail -2
done
