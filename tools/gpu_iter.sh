#!/bin/bash
# iteration loop on the GPU box: build, quick parity, benches, launch list.
# usage: bash tools/gpu_iter.sh [tag] [extra pytest -k expr]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-iter}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { cat gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q --durations=5 -k "${2:-not full_size and not c5a and not random_small}" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -3 gpurun_out/${TAG}_pytest.log
for W in C5B C3; do
  timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_bench_${W}.json 2> gpurun_out/${TAG}_bench_${W}.err
  python -c "import json,sys; d=json.load(open('gpurun_out/${TAG}_bench_${W}.json')); print('$W', round(d['ms_per_step'],2),'ms', '%.3g'%d['value'], {k:round(v,2) for k,v in d['stage_ms'].items()}, 'frac', round(d['roofline']['frac'],3))"
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c5b.csv python tools/one_build.py C5B 2 > /dev/null 2>&1
