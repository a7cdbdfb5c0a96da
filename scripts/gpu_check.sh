#!/bin/bash
TAG=${1:-r02h}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; tail -1 gpurun_out/${TAG}_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_gputest.txt 2>&1; grep -E "passed|failed" gpurun_out/${TAG}_gputest.txt | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cut -c1-300 gpurun_out/${TAG}_bench.json
timeout 900 python scripts/time_configs.py C1 C2 C3 P C4 C5 > gpurun_out/${TAG}_configs.txt 2>&1; cat gpurun_out/${TAG}_configs.txt
