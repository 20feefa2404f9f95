#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-proft}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_tets -s 2 -c 2 -o gpurun_out/${TAG} python tools/one_build.py C4 2 > gpurun_out/${TAG}_ncu.log 2>&1
tail -2 gpurun_out/${TAG}_ncu.log
