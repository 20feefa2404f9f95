#!/bin/bash
# bucket edge path: its tests, a C5A launch list of the k_bk kernels, C5A/C5B stage times
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-bq}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" >/dev/null 2>&1
timeout 600 python -m pytest tests/test_edge_buckets_gpu.py -q -x 2>&1 | tail -2
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv -k regex:"k_bk_|k_dist|k_gp" --log-file gpurun_out/${TAG}.csv python tools/one_build.py C5A 1 > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}.csv 1 2>&1 | head -4
for W in C5A C5B; do python bench.py --workload $W --steps 5 --warmup 3 --no-cpu-baseline --no-e2e 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$W', round(d['ms_per_step'],2), {k:round(v,2) for k,v in d['stage_ms'].items() if v})"; done
