#!/bin/bash
# Round-2 first GPU pass: smoke, full GPU suite, bench fp64 + fp32, fp32 report.
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r02a_smi.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02a_smoke.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -x --durations=15 > gpurun_out/r02a_gputest.txt 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r02a_bench.json 2> gpurun_out/r02a_bench.err
timeout 600 python bench.py --precision fp32 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r02a_bench_fp32.json 2> gpurun_out/r02a_bench_fp32.err
timeout 600 python scripts/fp32_report.py > gpurun_out/r02a_fp32_report.json 2>&1
tail -3 gpurun_out/r02a_gputest.txt
