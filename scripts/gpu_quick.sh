mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/q_all.log 2>&1; tail -5 gpurun_out/q_all.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"fold" python scripts/profile_once.py C3 2 > gpurun_out/dram_fold.csv 2>&1
grep fold gpurun_out/dram_fold.csv | cut -d, -f5,13-15 | head -12
timeout 300 python scripts/time_configs.py C3 P C4 > gpurun_out/q_time.log 2>&1; tail -3 gpurun_out/q_time.log
