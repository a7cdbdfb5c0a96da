mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "adversarial_inputs_fp32" > gpurun_out/q.log 2>&1; tail -25 gpurun_out/q.log
