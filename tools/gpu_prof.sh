#!/bin/bash
# ncu --set full capture of the triangle kernels (args: tag workload [npts])
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-prof}; W=${2:-C5B}; NP=${3:-}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || exit 1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_triangles -s 2 -c 2 -o gpurun_out/${TAG} python tools/one_build.py $W 2 $NP > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
tail -3 gpurun_out/${TAG}_ncu.log
