mkdir -p gpurun_out
timeout 300 python scripts/time_configs.py C3 P C4 C2 > gpurun_out/q_time.log 2>&1; tail -4 gpurun_out/q_time.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_all.log 2>&1; tail -4 gpurun_out/q_all.log
