#!/bin/bash
# round-2 evidence: ncu --set full of the C5B count + fill, C4 tetrahedron fill, C5A onesweep;
# DFMA counts of the distance kernels; the launch list of one C5B build.  usage: bash tools/gpu_prof_r2.sh tag
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-r2p}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
# launch list of the bench's C5B step (serialised, cold caches: shares, not absolute times)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_C5B.csv python tools/one_build.py C5B 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_launches_C5B.csv 2 > gpurun_out/${TAG}_launches_C5B.txt 2>&1
head -12 gpurun_out/${TAG}_launches_C5B.txt
# DFMA / DADD / DMUL executed by the distance kernels (C5B)
timeout 600 ncu --metrics gpu__time_duration.sum,sm__sass_thread_inst_executed_op_dfma_pred_on.sum,sm__sass_thread_inst_executed_op_dadd_pred_on.sum,sm__sass_thread_inst_executed_op_dmul_pred_on.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_dist --csv --log-file gpurun_out/${TAG}_dist_C5B.csv python tools/one_build.py C5B 1 > /dev/null 2>&1
echo "dist rc=$?"
# full sets: count + fill (C5B), tetrahedron fill (C4), one onesweep pass (C5A)
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_triangles -s 2 -c 2 -o gpurun_out/${TAG}_tri python tools/one_build.py C5B 2 > gpurun_out/${TAG}_tri.log 2>&1
echo "tri rc=$?"
{ python tools/ncu_summary.py gpurun_out/${TAG}_tri.ncu-rep "" 10; python tools/ncu_lines.py gpurun_out/${TAG}_tri.ncu-rep "k_triangles<(bool)1" 25; python tools/ncu_lines.py gpurun_out/${TAG}_tri.ncu-rep "k_triangles<(bool)0" 25; } > gpurun_out/${TAG}_ncu_tri_c5b.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tets_dense -s 1 -c 1 -o gpurun_out/${TAG}_tets python tools/one_build.py C4 1 > gpurun_out/${TAG}_tets.log 2>&1
echo "tets rc=$?"
{ python tools/ncu_summary.py gpurun_out/${TAG}_tets.ncu-rep "" 10; python tools/ncu_lines.py gpurun_out/${TAG}_tets.ncu-rep "k_tets_dense" 25; } > gpurun_out/${TAG}_ncu_tets_c4.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_onesweep -s 1 -c 1 -o gpurun_out/${TAG}_sweep python tools/one_build.py C5A 1 > gpurun_out/${TAG}_sweep.log 2>&1
echo "sweep rc=$?"
{ python tools/ncu_summary.py gpurun_out/${TAG}_sweep.ncu-rep "" 10; python tools/ncu_lines.py gpurun_out/${TAG}_sweep.ncu-rep "k_onesweep" 25; } > gpurun_out/${TAG}_ncu_sweep_c5a.txt 2>&1
rm -f gpurun_out/${TAG}_*.ncu-rep.tmp
ls -la gpurun_out/${TAG}_*
