# one optimisation iteration: parity, bench, ncu of the band kernel on a C3 prefix
TAG=${1:-it}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_${TAG}.log 2>&1; tail -3 gpurun_out/pytest_${TAG}.log
grep -E "AssertionError|Error" gpurun_out/pytest_${TAG}.log | head -5
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err; tail -2 gpurun_out/bench_${TAG}.err
python -c "import json;d=json.load(open('gpurun_out/bench_${TAG}.json'));print('value',d['value'],'ms',d['ms_per_step'],'frac',d['roofline']['frac'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sym_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG} python scripts/profile_once.py C3 2 393218 > gpurun_out/prof_${TAG}.log 2>&1
tail -1 gpurun_out/prof_${TAG}.log
