#!/bin/bash
# C5A launch list (edge ranking) + markfill C5B bench
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-c5a}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_C5A.csv python tools/one_build.py C5A 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_launches_C5A.csv 2 > gpurun_out/${TAG}_launches_C5A.txt 2>&1
cat gpurun_out/${TAG}_launches_C5A.txt | head -30


