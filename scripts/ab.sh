# A/B the band kernel of two library builds on the same box: bash scripts/ab.sh WORKLOAD
WL=${1:-C3}
for i in 1 2; do
for v in old new; do
  RQA_LIB_PATH=abtest/lib_$v.so timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ab_$v.csv python scripts/time_configs.py $WL > /dev/null 2>&1
  echo "$v $(grep -E 'unit_kernel|sym_kernel' gpurun_out/ab_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | head -1) $(grep -E 'fold' gpurun_out/ab_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | head -2 | tr '\n' ' ')"
done
done
