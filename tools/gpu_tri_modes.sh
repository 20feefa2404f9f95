#!/bin/bash
# C5B / C3 triangle stage under the three bitmap modes, plus the CUB sort calibration
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-modes}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
for W in C5B C3; do
  for M in pos rank none; do
    if [ $M = none ]; then export VRB_NO_APEX_BITMAPS=1; unset VRB_TRI_BITMAPS; else unset VRB_NO_APEX_BITMAPS; export VRB_TRI_BITMAPS=$M; fi
    timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${W}_${M}.json 2> gpurun_out/${TAG}_${W}_${M}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${W}_${M}.json')); print('$W $M', round(d['ms_per_step'],2),'ms', {k:round(v,2) for k,v in d['stage_ms'].items() if v})" || tail -3 gpurun_out/${TAG}_${W}_${M}.err
  done
done
unset VRB_NO_APEX_BITMAPS VRB_TRI_BITMAPS
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a tools/calib/cub_sort.cu -o /tmp/cub_sort && /tmp/cub_sort 200000000 | tee gpurun_out/${TAG}_cub.txt
