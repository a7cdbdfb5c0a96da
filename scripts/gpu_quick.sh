mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tiny or largest" > gpurun_out/q_edge.log 2>&1; tail -15 gpurun_out/q_edge.log
