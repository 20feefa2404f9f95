#!/bin/bash
# round-end record: build + smoke, every GPU test, the default bench line (e2e + cpu_baseline),
# the other workloads' lines, the reference arm.  usage: bash tools/gpu_final.sh tag
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-final}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/${TAG}_gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest tests -m gpu -q --durations=10 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/${TAG}_pytest.log
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.json 2> gpurun_out/${TAG}_bench_default.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench_default.json
for W in C3 C4 C5A HIV; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 > gpurun_out/${TAG}_bench_${W}.json 2> gpurun_out/${TAG}_bench_${W}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${W}.json')); print('$W', round(d['ms_per_step'],2),'ms', '%.3g'%d['value'], {k:round(v,2) for k,v in d['stage_ms'].items() if v})" || tail -3 gpurun_out/${TAG}_bench_${W}.err
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/${TAG}_bench_reference.json 2>&1; tail -c 600 gpurun_out/${TAG}_bench_reference.json
