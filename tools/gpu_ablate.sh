#!/bin/bash
# fill ablation per variant: VRB_DEBUG_FILL=0 (full), 2 (no flush), 1 (mark only); C5B fill ms
# usage: bash tools/gpu_ablate.sh tag W name1 name2 ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; W=$2; shift 2
mkdir -p gpurun_out
for V in "$@"; do
  export VRB_LIB_PATH=$PWD/variants/$V/libvrb.so
  for D in 0 2 1; do
    VRB_DEBUG_FILL=$D timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${V}_${D}.json 2> gpurun_out/${TAG}_${V}_${D}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${V}_${D}.json')); print('$V debug=$D', 'fill', round(d['stage_ms']['fill'],2), 'count', round(d['stage_ms']['count'],2))" || tail -3 gpurun_out/${TAG}_${V}_${D}.err
  done
done
