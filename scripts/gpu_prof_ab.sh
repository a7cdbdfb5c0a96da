# ncu --set full of the unit kernel, float64 path vs f32 filter, C3 prefix
PRE=${1:-262146}
mkdir -p gpurun_out
RQA_FILTER=0 timeout 900 ncu --set full --clock-control none --import-source on -k regex:unit_kernel -s 1 -c 1 -o gpurun_out/prof_fp64 python scripts/profile_once.py C3 2 $PRE > gpurun_out/prof_fp64.log 2>&1
RQA_FILTER=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:unit_kernel -s 1 -c 1 -o gpurun_out/prof_f32 python scripts/profile_once.py C3 2 $PRE > gpurun_out/prof_f32.log 2>&1
tail -1 gpurun_out/prof_fp64.log gpurun_out/prof_f32.log
