#!/bin/bash
# round-2 third-session evidence: smoke, bench lines (all workloads), the
# reference arm, in-pipeline launch lists (ncu application replay), ncu
# --set full of the S3 bucket kernels on C5A.   usage: bash tools/gpu_round2s3.sh tag
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-r2s3}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench rc=$?"
for W in C3 C4 C5A HIV; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_${W}.json 2> gpurun_out/${TAG}_bench_${W}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${W}.json')); print('$W', round(d['ms_per_step'],2),'ms', '%.3g'%d['value'], d.get('edge_path'), {k:round(v,2) for k,v in d['stage_ms'].items() if v})" || tail -3 gpurun_out/${TAG}_bench_${W}.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1; tail -c 300 gpurun_out/${TAG}_bench_reference.json; echo
for W in C5B C5A; do
  timeout 900 ncu --replay-mode application --cache-control none --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --csv --log-file gpurun_out/${TAG}_inpipeline_${W}.csv python tools/one_build.py $W 2 > /dev/null 2>&1
  python tools/launches.py gpurun_out/${TAG}_inpipeline_${W}.csv 2 > gpurun_out/${TAG}_inpipeline_${W}.txt 2>&1
done
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_bk_|k_dist_full" -c 8 -o gpurun_out/${TAG}_bk python tools/one_build.py C5A 1 > /dev/null 2>&1
{ python tools/ncu_summary.py gpurun_out/${TAG}_bk.ncu-rep "" 10; python tools/ncu_lines.py gpurun_out/${TAG}_bk.ncu-rep "k_bk_rank" 25; python tools/ncu_lines.py gpurun_out/${TAG}_bk.ncu-rep "k_bk_scatter" 12; } > gpurun_out/${TAG}_ncu_bk_c5a.txt 2>&1
rm -f gpurun_out/${TAG}_*.ncu-rep
ls gpurun_out/${TAG}_*
