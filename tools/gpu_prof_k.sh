#!/bin/bash
# launch list (gpu__time_duration per kernel) of one build + ncu --set full of one kernel
# usage: bash tools/gpu_prof_k.sh tag workload kernel_regex launch_skip
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; W=$2; K=$3; SKIP=${4:-0}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv python tools/one_build.py $W 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_launches.csv 2 | head -20
if [ -n "$K" ]; then
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s $SKIP -c 1 -o gpurun_out/${TAG} python tools/one_build.py $W 1 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
fi
