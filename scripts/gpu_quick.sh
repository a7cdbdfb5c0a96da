timeout 300 python scripts/e2e_probe.py 2>&1 | tail -5
RQA_PREFILTER=0 timeout 300 python scripts/e2e_probe.py 2>&1 | tail -2
