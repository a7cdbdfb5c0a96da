# ncu --set full of the full-size C3 unit kernel (traffic for bench.py) + 2-rank shared-GPU bench
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:unit_kernel -s 1 -c 1 -o gpurun_out/prof_C3full python scripts/profile_once.py C3 2 > gpurun_out/prof_C3full.log 2>&1
tail -1 gpurun_out/prof_C3full.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"unit_kernel|fold" python scripts/profile_once.py C3 2 > gpurun_out/dram_C3.csv 2>&1
bash scripts/gpu_multi.sh
