mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv -k regex:"fold" python scripts/profile_once.py C3 2 > gpurun_out/fold_t.csv 2>&1
grep fold gpurun_out/fold_t.csv | python3 -c "
import csv,sys
for r in csv.reader(sys.stdin): print(r[4][:20], r[-1])"
