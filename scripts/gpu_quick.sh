mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_precision.py -x -q -k "stripes" > gpurun_out/q.log 2>&1; tail -3 gpurun_out/q.log
