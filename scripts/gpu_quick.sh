# quick GPU check: precision tests + parity tests + short C3 timing both paths
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precision.py -x -q > gpurun_out/q_prec.log 2>&1; tail -15 gpurun_out/q_prec.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/q_all.log 2>&1; tail -5 gpurun_out/q_all.log
timeout 300 python scripts/time_configs.py C3 > gpurun_out/q_time_filter.log 2>&1; tail -3 gpurun_out/q_time_filter.log
RQA_FILTER=0 timeout 300 python scripts/time_configs.py C3 > gpurun_out/q_time_fp64.log 2>&1; tail -3 gpurun_out/q_time_fp64.log
