timeout 900 python scripts/fuzz_parity.py 2000 80 2>&1 | tail -1 | cut -c1-200
RQA_PREFILTER=1 timeout 900 python scripts/fuzz_parity.py 1000 81 2>&1 | tail -1 | cut -c1-200
timeout 600 python scripts/time_configs.py 2>&1 | cut -c1-80
