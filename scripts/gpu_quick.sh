mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_operators.py -x -q > gpurun_out/q_new.log 2>&1; tail -15 gpurun_out/q_new.log
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/q_all.log 2>&1; tail -5 gpurun_out/q_all.log
