# smoke + parity tests + bench + reference arm + launch list + ncu --set full (full C3)
TAG=${1:-r01d}
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; tail -1 gpurun_out/smoke_${TAG}.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/pytest_${TAG}.log 2>&1; tail -1 gpurun_out/pytest_${TAG}.log
timeout 600 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -1 gpurun_out/bench_${TAG}.err; cut -c1-300 gpurun_out/bench_${TAG}.json
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_${TAG}.json 2>&1; tail -1 gpurun_out/bench_ref_${TAG}.json | cut -c1-200
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"unit_kernel|fold" -s 3 -c 3 -o gpurun_out/prof_full_${TAG} python scripts/profile_once.py C3 2 > gpurun_out/prof_full_${TAG}.log 2>&1
tail -1 gpurun_out/prof_full_${TAG}.log
timeout 900 python scripts/stripe_projection.py C3 > gpurun_out/proj_${TAG}.log 2>&1; tail -1 gpurun_out/proj_${TAG}.log | cut -c1-200
