#!/bin/bash
# instructions of the bitmap count + fill on C3 and C5B (per-edge vs per-triangle cost split)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-fi}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for W in C3 C5B; do
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum,smsp__thread_inst_executed.sum --clock-control none -k regex:k_triangles --csv --log-file gpurun_out/${TAG}_${W}.csv python tools/one_build.py $W 1 > /dev/null 2>&1
grep -E "k_triangles" gpurun_out/${TAG}_${W}.csv | awk -F'","' '{print $5, $(NF-2), $(NF)}' | cut -c1-200
done
