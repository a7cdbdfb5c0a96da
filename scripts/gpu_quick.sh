# quick GPU check: new tests first, then the whole GPU suite, then short C3 timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_gpu_precision.py -x -q > gpurun_out/q_new.log 2>&1; tail -15 gpurun_out/q_new.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/q_all.log 2>&1; tail -5 gpurun_out/q_all.log
timeout 300 python scripts/time_configs.py C3 > gpurun_out/q_time.log 2>&1; tail -3 gpurun_out/q_time.log
