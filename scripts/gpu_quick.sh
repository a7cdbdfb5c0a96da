mkdir -p gpurun_out
timeout 1500 python scripts/fuzz_parity.py 4000 7 > gpurun_out/fuzz.log 2>&1; tail -1 gpurun_out/fuzz.log | cut -c1-400; cp gpurun_out/fuzz_parity.json gpurun_out/fuzz_parity_default.json
RQA_PREFILTER=1 timeout 1500 python scripts/fuzz_parity.py 2000 8 > gpurun_out/fuzz1.log 2>&1; tail -1 gpurun_out/fuzz1.log | cut -c1-400; cp gpurun_out/fuzz_parity.json gpurun_out/fuzz_parity_prefilter.json
RQA_FILTER=2 timeout 1500 python scripts/fuzz_parity.py 2000 9 > gpurun_out/fuzz2.log 2>&1; tail -1 gpurun_out/fuzz2.log | cut -c1-400; cp gpurun_out/fuzz_parity.json gpurun_out/fuzz_parity_f32filter.json
