mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_all.log 2>&1; tail -4 gpurun_out/q_all.log
timeout 300 python scripts/time_configs.py C3 > gpurun_out/q_time.log 2>&1; tail -1 gpurun_out/q_time.log
RQA_PREFILTER=0 timeout 300 python scripts/time_configs.py C3 > gpurun_out/q_time0.log 2>&1; tail -1 gpurun_out/q_time0.log
RQA_PREFILTER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:unit_kernel -s 1 -c 1 -o gpurun_out/prof_pre python scripts/profile_once.py C3 2 262146 > gpurun_out/prof_pre.log 2>&1; tail -1 gpurun_out/prof_pre.log
