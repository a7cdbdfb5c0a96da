mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_C3.csv python scripts/profile_once.py C3 2 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:band_kernel -s 1 -c 1 -o gpurun_out/prof_C3 python scripts/profile_once.py C3 2 > gpurun_out/prof_C3.log 2>&1
tail -3 gpurun_out/prof_C3.log
ls -la gpurun_out
