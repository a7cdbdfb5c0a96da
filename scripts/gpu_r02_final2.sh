#!/bin/bash
# Round-2 closing evidence on the final build: smoke, GPU suite, bench (fp64 +
# reference arm + fp32), config timings, launch list + ncu of C3 / C4 / P,
# the checked build (bounds assertions; compute-sanitizer is closed on this
# pool), stress fuzz.  Build the checked library first:
# EXTRA=-DRQA_CHECKS bash scripts/ab_build.sh checked
TAG=${1:-r02z}
cd "$GRAFT_REPO_ROOT"; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/${TAG}_smi.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.txt 2>&1; tail -1 gpurun_out/${TAG}_smoke.txt
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > gpurun_out/${TAG}_gputest.txt 2>&1; grep -E "passed|failed" gpurun_out/${TAG}_gputest.txt | tail -1
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; cut -c1-200 gpurun_out/${TAG}_bench.json
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_bench_ref.json 2>&1; cut -c1-160 gpurun_out/${TAG}_bench_ref.json
timeout 900 python bench.py --precision fp32 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_fp32.json 2> gpurun_out/${TAG}_bench_fp32.err; cut -c1-160 gpurun_out/${TAG}_bench_fp32.json
timeout 900 python scripts/time_configs.py C1 C2 C3 P C4 C5 > gpurun_out/${TAG}_configs.txt 2>&1; cat gpurun_out/${TAG}_configs.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
for W in C3 C4 P; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"unit_kernel" -s 1 -c 1 \
    -o gpurun_out/${TAG}_ncu_$W python scripts/profile_once.py $W 2 > gpurun_out/${TAG}_ncu_$W.log 2>&1; tail -1 gpurun_out/${TAG}_ncu_$W.log
done
timeout 900 ncu --set full --clock-control none -k regex:"unit_fold_all" -c 1 -o gpurun_out/${TAG}_ncu_fold_C3 python scripts/profile_once.py C3 1 > gpurun_out/${TAG}_ncu_fold.log 2>&1; tail -1 gpurun_out/${TAG}_ncu_fold.log
# compute-sanitizer is closed on this GPU pool: the checked build (device
# bounds / capacity assertions, scripts/gpu_checked.sh) stands in for it
[ -f abtest/checked/librqa_b200.so ] && bash scripts/gpu_checked.sh ${TAG}
(RQA_FLUSH_EVERY=2 RQA_MIN_UNIT=4 timeout 600 python scripts/fuzz_parity.py 400 101 12000; RQA_FLUSH_EVERY=4 RQA_PREFILTER=1 RQA_WAVES=64 timeout 600 python scripts/fuzz_parity.py 400 202 20000; timeout 900 python scripts/fuzz_parity.py 600 404 30000) > gpurun_out/${TAG}_fuzz.txt 2>&1; grep cases gpurun_out/${TAG}_fuzz.txt
