#!/bin/bash
# in-pipeline launch list (ncu application replay, no cache flush): per-kernel
# times as they run inside a build, not serialised cold-cache replays
# usage: bash tools/gpu_launches_app.sh tag "C5B C5A"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-app}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for W in ${2:-C5B}; do
  timeout 900 ncu --replay-mode application --cache-control none --clock-control none --metrics gpu__time_duration.sum --csv --log-file gpurun_out/${TAG}_launches_${W}.csv python tools/one_build.py $W 2 > /dev/null 2>&1
  python tools/launches.py gpurun_out/${TAG}_launches_${W}.csv 2 > gpurun_out/${TAG}_launches_${W}.txt 2>&1
  echo "== $W"; head -25 gpurun_out/${TAG}_launches_${W}.txt
done
