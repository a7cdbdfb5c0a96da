mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_all.log 2>&1; tail -2 gpurun_out/q_all.log
timeout 300 python scripts/e2e_probe.py 2>&1 | tail -3
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err; python -c "
import json; d=json.load(open('gpurun_out/b.json')); print(d['value'], d['e2e']['value'], d['full_rqa'])"
