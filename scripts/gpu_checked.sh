#!/bin/bash
# Checked build (device bounds / capacity assertions, make EXTRA=-DRQA_CHECKS,
# built by scripts/ab_build.sh checked) over the GPU suite, the sanitizer case
# list with the mid-unit flush path, and a fuzz sweep.  Stands in for
# compute-sanitizer, which this GPU pool no longer allows.
TAG=${1:-r02c}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
export RQA_LIB_PATH=$PWD/abtest/checked/librqa_b200.so
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/${TAG}_checked_gputest.txt 2>&1; echo "gputest rc=$?"; grep -E "passed|failed|RQA_DCHECK" gpurun_out/${TAG}_checked_gputest.txt | tail -3
RQA_PREFILTER=1 RQA_FLUSH_EVERY=2 timeout 900 python scripts/sanitize_cases.py 1200 > gpurun_out/${TAG}_checked_cases.txt 2>&1; echo "cases rc=$?"; tail -2 gpurun_out/${TAG}_checked_cases.txt
(RQA_FLUSH_EVERY=2 RQA_MIN_UNIT=4 timeout 600 python scripts/fuzz_parity.py 300 707 12000; RQA_PREFILTER=1 RQA_WAVES=64 timeout 600 python scripts/fuzz_parity.py 300 808 20000) > gpurun_out/${TAG}_checked_fuzz.txt 2>&1; echo "fuzz rc=$?"; grep -E "cases|DCHECK" gpurun_out/${TAG}_checked_fuzz.txt | cut -c1-200
