mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/q_all.log 2>&1; tail -2 gpurun_out/q_all.log
