mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"fold" python scripts/profile_once.py C3 2 > gpurun_out/fold_t.csv 2>&1
grep fold gpurun_out/fold_t.csv | cut -d, -f5,15 | head -4
timeout 300 python scripts/time_configs.py C3 > gpurun_out/q_time.log 2>&1; tail -1 gpurun_out/q_time.log
