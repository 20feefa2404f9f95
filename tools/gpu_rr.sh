#!/bin/bash
# rank-ordered-records triangle path: parity + C5B/C3 bench lines vs the default path
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-rr}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || { tail gpurun_out/${TAG}_build.log; exit 1; }
timeout 900 python -m pytest tests/test_parity_gpu.py -q -x -k "path_variants or c1 or c2" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 600 python -m pytest tests/test_h0_gpu.py -q -x -k compress > gpurun_out/${TAG}_pytest_h0.log 2>&1; echo "pytest h0 rc=$?"; tail -2 gpurun_out/${TAG}_pytest_h0.log
for W in C5B C3; do
  for P in bitmap xmajor; do
    VRB_TRI_PATH=$P timeout 600 python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_${W}_${P}.json 2> gpurun_out/${TAG}_${W}_${P}.err
    python -c "import json; d=json.load(open('gpurun_out/${TAG}_${W}_${P}.json')); print('$W $P', round(d['ms_per_step'],2),'ms', '%.3g'%d['value'], {k:round(v,2) for k,v in d['stage_ms'].items() if v}, d.get('h0_barcodes',{}).get('clear_compress',{}).get('ms'))" || tail -3 gpurun_out/${TAG}_${W}_${P}.err
  done
done
