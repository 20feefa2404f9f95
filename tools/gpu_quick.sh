#!/bin/bash
# quick iteration: build, all GPU tests, C5B/C3 (+ optional extra workloads) bench lines
# usage: bash tools/gpu_quick.sh tag [workloads...]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-q}; shift
WLS=${@:-C5B C3}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { cat gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -4 gpurun_out/${TAG}_pytest.log
for W in $WLS; do
  timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_${W}.json 2> gpurun_out/${TAG}_bench_${W}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${W}.json')); print('$W', round(d['ms_per_step'],2),'ms', '%.3g'%d['value'], {k:round(v,2) for k,v in d['stage_ms'].items()})" || tail -5 gpurun_out/${TAG}_bench_${W}.err
done
