#!/bin/bash
# compute-sanitizer (memcheck / racecheck / synccheck / initcheck) over tools/sanitize_run.py
# usage: bash tools/gpu_sanitize.sh tag
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-san}
mkdir -p gpurun_out/${TAG}
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
for T in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $T --target-processes all python tools/sanitize_run.py > gpurun_out/${TAG}/$T.txt 2>&1
  echo "$T rc=$? $(tail -1 gpurun_out/${TAG}/$T.txt)"
done
