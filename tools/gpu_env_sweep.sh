#!/bin/bash
# bench one workload under several values of an environment knob
# usage: bash tools/gpu_env_sweep.sh tag VAR "v1 v2 ..." "W1 W2"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; VAR=$2; VALS=$3; WS=$4
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for W in $WS; do
  for V in $VALS; do
    env $VAR=$V timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${W}_${V}.json 2> gpurun_out/${TAG}_${W}_${V}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${W}_${V}.json')); print('$W $VAR=$V', round(d['ms_per_step'],2),'ms', {k:round(v,2) for k,v in d['stage_ms'].items() if v})" || tail -3 gpurun_out/${TAG}_${W}_${V}.err
  done
done
