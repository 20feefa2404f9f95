#!/bin/bash
# round-2 second-session evidence: bench lines (all workloads), in-pipeline launch lists
# (ncu application replay), ncu --set full of the C5B count + fill, C5A onesweep + k_rank_edges,
# C4 tetrahedron fill, HIV keys-only onesweep.   usage: bash tools/gpu_round2s2.sh tag
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-r2s2}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench rc=$?"
for W in C3 C4 C5A HIV; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_${W}.json 2> gpurun_out/${TAG}_bench_${W}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${W}.json')); print('$W', round(d['ms_per_step'],2),'ms', '%.3g'%d['value'], {k:round(v,2) for k,v in d['stage_ms'].items() if v})" || tail -3 gpurun_out/${TAG}_bench_${W}.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1; tail -c 300 gpurun_out/${TAG}_bench_reference.json; echo
for W in C5B C5A C4 HIV; do
  timeout 900 ncu --replay-mode application --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/${TAG}_inpipeline_${W}.csv python tools/one_build.py $W 2 > /dev/null 2>&1
  python tools/launches.py gpurun_out/${TAG}_inpipeline_${W}.csv 2 > gpurun_out/${TAG}_inpipeline_${W}.txt 2>&1
done
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_triangles -s 2 -c 2 -o gpurun_out/${TAG}_tri python tools/one_build.py C5B 2 > /dev/null 2>&1
{ python tools/ncu_summary.py gpurun_out/${TAG}_tri.ncu-rep "" 10; python tools/ncu_lines.py gpurun_out/${TAG}_tri.ncu-rep "k_triangles" 30; } > gpurun_out/${TAG}_ncu_tri_c5b.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_onesweep|k_rank_edges|k_dist_full" -s 0 -c 6 -o gpurun_out/${TAG}_c5a python tools/one_build.py C5A 1 > /dev/null 2>&1
{ python tools/ncu_summary.py gpurun_out/${TAG}_c5a.ncu-rep "" 10; python tools/ncu_lines.py gpurun_out/${TAG}_c5a.ncu-rep "k_rank_edges" 20; } > gpurun_out/${TAG}_ncu_c5a.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tets_dense -s 1 -c 1 -o gpurun_out/${TAG}_tets python tools/one_build.py C4 1 > /dev/null 2>&1
{ python tools/ncu_summary.py gpurun_out/${TAG}_tets.ncu-rep "" 10; python tools/ncu_lines.py gpurun_out/${TAG}_tets.ncu-rep "k_tets_dense" 20; } > gpurun_out/${TAG}_ncu_tets_c4.txt 2>&1
rm -f gpurun_out/${TAG}_*.ncu-rep
ls gpurun_out/${TAG}_*
