#!/bin/bash
# compare experiment builds (variants/<name>/libvrb.so): full-size C5B parity + bench lines
# usage: bash tools/gpu_variants.sh tag "C5B C3" name1 name2 ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; WLS=$2; shift 2
mkdir -p gpurun_out
for V in "$@"; do
  export VRB_LIB_PATH=$PWD/variants/$V/libvrb.so
  timeout 600 python -m pytest tests -m gpu -x -q -k "${PYK:-full_size_config and (C5B or C3 or C4) or golden or random}" > gpurun_out/${TAG}_${V}_pytest.log 2>&1
  echo "$V pytest: $(tail -1 gpurun_out/${TAG}_${V}_pytest.log)"
  for W in $WLS; do
    timeout 600 python bench.py --workload $W --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${V}_${W}.json 2> gpurun_out/${TAG}_${V}_${W}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${V}_${W}.json')); print('  $V $W', round(d['ms_per_step'],2),'ms', {k:round(v,2) for k,v in d['stage_ms'].items() if v})" || tail -3 gpurun_out/${TAG}_${V}_${W}.err
  done
done
