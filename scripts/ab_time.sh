#!/bin/bash
# Interleaved timing of A/B variants: VARIANTS="base x y" WLS="C3 C4" ROUNDS=2
cd "$GRAFT_REPO_ROOT"
for r in $(seq ${ROUNDS:-2}); do
  for v in ${VARIANTS}; do
    for w in ${WLS:-C3}; do
      echo -n "$v "; RQA_LIB_PATH=$PWD/abtest/$v/librqa_b200.so timeout 600 python scripts/time_configs.py $w 2>&1 | tail -1
    done
  done
done
