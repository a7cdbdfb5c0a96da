timeout 1500 python scripts/fuzz_parity.py 400 92 40000 > /dev/null 2>&1; cp gpurun_out/fuzz_parity.json gpurun_out/fz_a.json
RQA_PREFILTER=1 timeout 1500 python scripts/fuzz_parity.py 300 93 40000 > /dev/null 2>&1; cp gpurun_out/fuzz_parity.json gpurun_out/fz_b.json
RQA_FILTER=2 timeout 1500 python scripts/fuzz_parity.py 300 94 40000 > /dev/null 2>&1; cp gpurun_out/fuzz_parity.json gpurun_out/fz_c.json
timeout 1500 python scripts/fuzz_parity.py 4000 95 6000 > /dev/null 2>&1; cp gpurun_out/fuzz_parity.json gpurun_out/fz_d.json
