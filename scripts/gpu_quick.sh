#!/bin/bash
# Quick check: GPU parity subset + config timings + launch list of one C3 run.
TAG=${1:-q}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full.py tests/test_gpu_multi.py -q -x > gpurun_out/${TAG}_pytest.txt 2>&1
tail -2 gpurun_out/${TAG}_pytest.txt
timeout 900 python scripts/time_configs.py ${CONFIGS:-C3 C4 P C2} > gpurun_out/${TAG}_configs.txt 2>&1
cat gpurun_out/${TAG}_configs.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python scripts/profile_once.py ${WL:-C3} 1 > /dev/null 2>&1
grep -o '"[a-z_:]*\(unit_kernel\|fold\|fix_diag\)[^"]*","[^"]*","[^"]*","[^"]*","[^"]*"' gpurun_out/${TAG}_launches.csv | cut -c1-40 | head; python - << 'PY'
import csv,sys
for r in csv.DictReader(l for l in open(f"gpurun_out/${TAG}_launches.csv") if not l.startswith("==")):
    print(r["Kernel Name"][:50], r["Metric Unit"], r["Metric Value"])
PY
