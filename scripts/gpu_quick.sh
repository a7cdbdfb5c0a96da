mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/b.json 2> gpurun_out/b.err; tail -2 gpurun_out/b.err; cat gpurun_out/b.json
timeout 600 python scripts/time_configs.py > gpurun_out/q_time.log 2>&1; tail -6 gpurun_out/q_time.log
