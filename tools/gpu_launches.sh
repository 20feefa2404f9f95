#!/bin/bash
# ncu launch list (gpu__time_duration, clocks not locked) of N builds of a workload; summary of the last
# usage: bash tools/gpu_launches.sh tag W [reps]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; W=$2; R=${3:-2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_${W}.csv python tools/one_build.py $W $R > gpurun_out/${TAG}_launches_${W}.log 2>&1
python tools/launches.py gpurun_out/${TAG}_launches_${W}.csv $R > gpurun_out/${TAG}_launches_${W}.txt 2>&1
head -25 gpurun_out/${TAG}_launches_${W}.txt
