#!/bin/bash
# ncu --set full of the triangle count + fill kernels (second build) and an e2e bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-pf}; W=${2:-C5B}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || exit 1
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench.json 2>&1
python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench.json')); print(round(d['ms_per_step'],2), 'e2e', d['e2e'])"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_triangles -s 2 -c 2 -o gpurun_out/${TAG} python tools/one_build.py $W 2 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"; tail -2 gpurun_out/${TAG}_ncu.log
