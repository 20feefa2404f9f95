#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-tet}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1 || exit 1
timeout 900 python -m pytest tests -m gpu -x -q -k "tetra or c2 or c4" > gpurun_out/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
tail -2 gpurun_out/${TAG}_pytest.log
timeout 600 python tools/time_stages.py C4 3
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches_c4.csv python tools/one_build.py C4 2 > /dev/null 2>&1
python tools/launches.py gpurun_out/${TAG}_launches_c4.csv 2>/dev/null | head -6
