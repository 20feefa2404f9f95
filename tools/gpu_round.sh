#!/bin/bash
# full round check on the GPU box: build, smoke, all GPU tests, default bench
# line (with e2e + cpu_baseline), C3/C4 bench lines, reference arm, C5B launch list.
# usage: bash tools/gpu_round.sh [tag]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-round}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/${TAG}_smoke.log
tail -2 gpurun_out/${TAG}_smoke.log
timeout 1200 python -m pytest tests -m gpu -x -q --durations=8 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench_default.json
for W in C3 C4 C5A; do
  timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_${W}.json 2> gpurun_out/${TAG}_bench_${W}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${W}.json')); print('$W', round(d['ms_per_step'],2),'ms', '%.3g'%d['value'], {k:round(v,2) for k,v in d['stage_ms'].items()})"
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1; tail -1 gpurun_out/${TAG}_bench_reference.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c5b.csv python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_launches_c5b.csv 4 2>/dev/null | head -14
# ncu --set full of the dominant kernel (the triangle fill) in the bench's launch configuration
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_triangles -s 2 -c 2 -o gpurun_out/${TAG}_fill python tools/one_build.py C5B 2 > gpurun_out/${TAG}_fill_ncu.log 2>&1
echo "ncu full rc=$?"
{ python tools/ncu_summary.py gpurun_out/${TAG}_fill.ncu-rep "" 8; python tools/ncu_lines.py gpurun_out/${TAG}_fill.ncu-rep "k_triangles<(bool)1" 40; } > gpurun_out/${TAG}_ncu_fill_c5b.txt 2>&1
# the C4 tetrahedron fill (its bench line names it)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tets_dense -s 1 -c 1 -o gpurun_out/${TAG}_tets python tools/one_build.py C4 1 > gpurun_out/${TAG}_tets_ncu.log 2>&1
{ python tools/ncu_summary.py gpurun_out/${TAG}_tets.ncu-rep "" 8; python tools/ncu_lines.py gpurun_out/${TAG}_tets.ncu-rep "k_tets_dense" 30; } > gpurun_out/${TAG}_ncu_tets_c4.txt 2>&1
head -5 gpurun_out/${TAG}_ncu_fill_c5b.txt
