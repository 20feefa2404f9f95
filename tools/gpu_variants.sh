#!/bin/bash
# bench a set of experiment builds (variants/<name>/libvrb.so) on workloads
# usage: bash tools/gpu_variants.sh tag "v1 v2 ..." "W1 W2 ..."
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; VS=$2; WS=$3
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for W in $WS; do
  for V in $VS; do
    VRB_LIB_PATH=variants/$V/libvrb.so timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${W}_${V}.json 2> gpurun_out/${TAG}_${W}_${V}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${W}_${V}.json')); print('$W $V', round(d['ms_per_step'],2),'ms', {k:round(v,2) for k,v in d['stage_ms'].items() if v})" || tail -3 gpurun_out/${TAG}_${W}_${V}.err
  done
done
