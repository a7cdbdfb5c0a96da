# ncu of the band kernel for a given geometry override on a C3 prefix
TAG=$1; GEOM=$2; PRE=${3:-606210}
mkdir -p gpurun_out
RQA_GEOMETRY=$GEOM timeout 600 ncu --set full --clock-control none --import-source on -k regex:"(sym|pipe)_kernel" -s 1 -c 1 -o gpurun_out/prof_${TAG} python scripts/profile_once.py C3 2 $PRE > gpurun_out/prof_${TAG}.log 2>&1
tail -1 gpurun_out/prof_${TAG}.log
