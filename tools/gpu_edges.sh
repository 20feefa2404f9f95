#!/bin/bash
# bucket edge path: its tests, the parity suite, stage times of the edge-heavy configs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-eb}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_edge_buckets_gpu.py -q -x > gpurun_out/${TAG}_eb.log 2>&1; echo "edge tests rc=$?"; tail -15 gpurun_out/${TAG}_eb.log
for W in C5A C5B C3 C4 HIV; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${W}.json 2> gpurun_out/${TAG}_${W}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_${W}.json')); print('$W', round(d['ms_per_step'],2),'ms', '%.3g'%d['value'], {k:round(v,2) for k,v in d['stage_ms'].items() if v})" || tail -3 gpurun_out/${TAG}_${W}.err
done
if [ "$2" = "full" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_gpu.log 2>&1; echo "gpu tests rc=$?"; tail -5 gpurun_out/${TAG}_gpu.log
fi
