#!/bin/bash
# quick GPU check: build, smoke, the named test files (or all -m gpu), one bench line
# usage: bash tools/gpu_check.sh tag "tests/test_a.py tests/test_b.py" [bench workloads...]
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-chk}; TESTS=${2:-tests}; shift 2
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/${TAG}_smoke.log
timeout 1500 python -m pytest $TESTS -m gpu -x -q --durations=10 > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/${TAG}_pytest.log
for W in "$@"; do
  timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_bench_${W}.json 2> gpurun_out/${TAG}_bench_${W}.err
  python -c "import json; d=json.load(open('gpurun_out/${TAG}_bench_${W}.json')); print('$W', round(d['ms_per_step'],2),'ms', '%.3g'%d['value'], {k:round(v,2) for k,v in d['stage_ms'].items()})" || tail -3 gpurun_out/${TAG}_bench_${W}.err
done
