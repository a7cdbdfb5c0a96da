#!/bin/bash
# One build->measure iteration: parity subset, config timings, forced-prefilter fuzz.
TAG=${1:-iter}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_precision.py tests/test_gpu_full.py -q -x > gpurun_out/${TAG}_pytest.txt 2>&1
tail -3 gpurun_out/${TAG}_pytest.txt
timeout 600 python scripts/time_configs.py ${CONFIGS:-C3 C4 P C2 C5} > gpurun_out/${TAG}_configs.txt 2>&1
cat gpurun_out/${TAG}_configs.txt
RQA_PREFILTER=1 timeout 600 python scripts/fuzz_parity.py ${FUZZ:-300} 7 8000 > gpurun_out/${TAG}_fuzz.txt 2>&1
tail -2 gpurun_out/${TAG}_fuzz.txt
