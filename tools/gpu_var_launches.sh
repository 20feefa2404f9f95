#!/bin/bash
# launch lists (gpu__time_duration) of one build per experiment variant
# usage: bash tools/gpu_var_launches.sh tag "v1 v2 ..." W [kernel-regex]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; VS=$2; W=$3; K=${4:-.}
mkdir -p gpurun_out
for V in $VS; do
  VRB_LIB_PATH=variants/$V/libvrb.so timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:$K --log-file gpurun_out/${TAG}_${V}.csv python tools/one_build.py $W 1 > gpurun_out/${TAG}_${V}.log 2>&1
  echo "== $V"; python tools/launches.py gpurun_out/${TAG}_${V}.csv 1 2>&1 | head -6
done
