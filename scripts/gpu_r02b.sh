#!/bin/bash
# Round-2 evidence pass: smoke, full GPU suite, bench (fp64, fp32, reference arm),
# launch list of the bench command, one ncu --set full of the C3 hot kernel.
TAG=${1:-r02b}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/${TAG}_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; tail -1 gpurun_out/${TAG}_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_gputest.txt 2>&1; tail -3 gpurun_out/${TAG}_gputest.txt
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cut -c1-600 gpurun_out/${TAG}_bench.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>&1; cut -c1-300 gpurun_out/${TAG}_bench_ref.json
timeout 600 python bench.py --precision fp32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_fp32.json 2> gpurun_out/${TAG}_bench_fp32.err; cut -c1-300 gpurun_out/${TAG}_bench_fp32.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"unit_kernel" -s 1 -c 1 \
  -o gpurun_out/${TAG}_ncu_C3full python scripts/profile_once.py C3 2 > gpurun_out/${TAG}_ncu_C3full.log 2>&1
tail -1 gpurun_out/${TAG}_ncu_C3full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"unit_kernel" -s 1 -c 1 \
  -o gpurun_out/${TAG}_ncu_C4full python scripts/profile_once.py C4 2 > gpurun_out/${TAG}_ncu_C4full.log 2>&1
tail -1 gpurun_out/${TAG}_ncu_C4full.log
