#!/bin/bash
# timelines (host gaps) + ncu --set full of the count kernel (C5B), one onesweep pass (C5A), the dense tet fill (C4)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/p3_build.log 2>&1 || exit 1
for W in C5B C4 C5A; do timeout 300 python tools/timeline.py $W 10 > gpurun_out/p3_tl_$W.txt 2>&1; tail -25 gpurun_out/p3_tl_$W.txt; done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_triangles -s 0 -c 1 -o gpurun_out/p3_count python tools/one_build.py C5B 1 > gpurun_out/p3_count.log 2>&1; echo "count rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 1 -c 1 -o gpurun_out/p3_sweep python tools/one_build.py C5A 1 > gpurun_out/p3_sweep.log 2>&1; echo "sweep rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tets_dense -s 1 -c 1 -o gpurun_out/p3_tets python tools/one_build.py C4 1 > gpurun_out/p3_tets.log 2>&1; echo "tets rc=$?"
ls -la gpurun_out/p3_*
