mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_all.log 2>&1; tail -2 gpurun_out/q_all.log
timeout 600 python scripts/time_configs.py > gpurun_out/q_time.log 2>&1; cat gpurun_out/q_time.log
timeout 900 python scripts/stripe_projection.py C3 > gpurun_out/proj.log 2>&1; tail -3 gpurun_out/proj.log | cut -c1-150
