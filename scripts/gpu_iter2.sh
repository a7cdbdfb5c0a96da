#!/bin/bash
# One build->measure iteration: full GPU suite, config timings, fuzz (default + forced prefilter).
TAG=${1:-iter}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.txt 2>&1
tail -3 gpurun_out/${TAG}_pytest.txt
timeout 900 python scripts/time_configs.py ${CONFIGS:-C3 C4 P C2 C5} > gpurun_out/${TAG}_configs.txt 2>&1
cat gpurun_out/${TAG}_configs.txt
timeout 600 python scripts/fuzz_parity.py ${FUZZ:-300} 11 8000 > gpurun_out/${TAG}_fuzz.txt 2>&1
tail -2 gpurun_out/${TAG}_fuzz.txt
RQA_PREFILTER=1 RQA_MIN_UNIT=4 timeout 600 python scripts/fuzz_parity.py ${FUZZ:-300} 7 8000 > gpurun_out/${TAG}_fuzz_pre.txt 2>&1
tail -2 gpurun_out/${TAG}_fuzz_pre.txt
