#!/bin/bash
# bench lines under different values of one env knob
# usage: bash tools/gpu_env_sweep.sh tag VAR "v1 v2 ..." "C5B C3"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; VAR=$2; VALS=$3; WLS=$4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || exit 1
for v in $VALS; do
  for W in $WLS; do
    env $VAR=$v timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${v}_${W}.json 2> gpurun_out/${TAG}_${v}_${W}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${v}_${W}.json')); print('$VAR=$v $W', round(d['ms_per_step'],2), {k:round(x,2) for k,x in d['stage_ms'].items() if x})" || tail -3 gpurun_out/${TAG}_${v}_${W}.err
  done
done
