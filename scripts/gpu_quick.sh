mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/q_all.log 2>&1; tail -1 gpurun_out/q_all.log
timeout 900 python scripts/fuzz_parity.py 1000 78 > gpurun_out/fuzz.log 2>&1; tail -1 gpurun_out/fuzz.log | cut -c1-200
