#!/bin/bash
# quick check: build, a test selection, bench lines of given workloads
# usage: bash tools/gpu_quick.sh tag "pytest -k expr" "C5B C5A ..."
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-q}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
if [ -n "$2" ]; then
  timeout 1200 python -m pytest tests -m gpu -q -x -k "$2" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
fi
for W in $3; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${W}.json 2> gpurun_out/${TAG}_${W}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_${W}.json')); print('$W', round(d['ms_per_step'],2),'ms', '%.3g'%d['value'], {k:round(v,2) for k,v in d['stage_ms'].items() if v})" || tail -3 gpurun_out/${TAG}_${W}.err
done
