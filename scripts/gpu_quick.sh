mkdir -p gpurun_out
for wl in P C4 C2; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:unit_kernel -s 1 -c 1 -o gpurun_out/prof_${wl} python scripts/profile_once.py $wl 2 > gpurun_out/prof_${wl}.log 2>&1; tail -1 gpurun_out/prof_${wl}.log
done
