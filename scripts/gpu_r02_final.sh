#!/bin/bash
# Round-2 evidence pass on the current build: smoke, GPU suite, bench (fp64 +
# reference arm + fp32), config timings, launch list + ncu --set full of the
# hot kernels, stripe projections, compute-sanitizer.
TAG=${1:-r02f}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; tail -1 gpurun_out/${TAG}_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_gputest.txt 2>&1; tail -2 gpurun_out/${TAG}_gputest.txt
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cut -c1-300 gpurun_out/${TAG}_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>&1; cut -c1-200 gpurun_out/${TAG}_bench_ref.json
timeout 900 python bench.py --precision fp32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_fp32.json 2> gpurun_out/${TAG}_bench_fp32.err; cut -c1-200 gpurun_out/${TAG}_bench_fp32.json
timeout 900 python scripts/time_configs.py C1 C2 C3 P C4 C5 > gpurun_out/${TAG}_configs.txt 2>&1; cat gpurun_out/${TAG}_configs.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for W in C3 C4 P; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"unit_kernel" -s 1 -c 1 \
    -o gpurun_out/${TAG}_ncu_$W python scripts/profile_once.py $W 2 > gpurun_out/${TAG}_ncu_$W.log 2>&1; tail -1 gpurun_out/${TAG}_ncu_$W.log
done
timeout 900 python scripts/stripe_projection.py C3 > gpurun_out/${TAG}_proj_C3.json 2> gpurun_out/${TAG}_proj_C3.err; tail -3 gpurun_out/${TAG}_proj_C3.json
timeout 1200 python scripts/stripe_projection.py C5 > gpurun_out/${TAG}_proj_C5.json 2> gpurun_out/${TAG}_proj_C5.err; tail -3 gpurun_out/${TAG}_proj_C5.json
export RQA_PREFILTER=1
for tool in memcheck synccheck initcheck racecheck; do
  timeout 1500 compute-sanitizer --tool $tool --print-limit 50 --error-exitcode 9 python scripts/sanitize_cases.py 1200 > gpurun_out/${TAG}_sanitize_${tool}.txt 2>&1
  echo "$tool rc=$?"; tail -1 gpurun_out/${TAG}_sanitize_${tool}.txt
done
