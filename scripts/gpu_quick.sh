mkdir -p gpurun_out
for k in 0 1 2 4 7; do echo "skip $k"; RQA_SKIP=$k timeout 300 python scripts/time_configs.py C3 2>&1 | tail -1 | cut -c1-60; done
