# usage: bash scripts/gpu_prof.sh TAG WORKLOAD PREFIX
TAG=${1:-sym}; WL=${2:-C3}; PRE=${3:-131074}
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv python scripts/profile_once.py $WL 2 $PRE > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sym_kernel -s 1 -c 1 -o gpurun_out/prof_${TAG} python scripts/profile_once.py $WL 2 $PRE > gpurun_out/prof_${TAG}.log 2>&1
tail -2 gpurun_out/prof_${TAG}.log
