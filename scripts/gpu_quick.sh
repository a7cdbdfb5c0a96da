mkdir -p gpurun_out
timeout 300 python scripts/time_configs.py C4 C3 > gpurun_out/q_time.log 2>&1; cat gpurun_out/q_time.log
RQA_PREFILTER=0 timeout 300 python scripts/time_configs.py C4 > gpurun_out/q_time0.log 2>&1; cat gpurun_out/q_time0.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_all.log 2>&1; tail -2 gpurun_out/q_all.log
