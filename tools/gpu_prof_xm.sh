#!/bin/bash
# ncu --set full of the x-major count + fill (C5B)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-xmp}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
export VRB_TRI_PATH=${2:-xmajor}
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_triangles|k_tri_fill" -s 2 -c 2 -o gpurun_out/${TAG}_tri python tools/one_build.py ${3:-C5B} 2 > gpurun_out/${TAG}_tri.log 2>&1
echo "tri rc=$?"
{ python tools/ncu_summary.py gpurun_out/${TAG}_tri.ncu-rep "" 10; python tools/ncu_lines.py gpurun_out/${TAG}_tri.ncu-rep "k_tri_fill" 30; python tools/ncu_lines.py gpurun_out/${TAG}_tri.ncu-rep "k_triangles" 25; } > gpurun_out/${TAG}_ncu_tri.txt 2>&1
