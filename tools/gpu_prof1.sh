#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c5b.csv python tools/one_build.py C5B 2 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_triangles -s 2 -c 2 -o gpurun_out/prof_tri_c5b10k python tools/one_build.py C5B 2 10000 > gpurun_out/ncu_full.log 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q -k "full_size or c5a" > gpurun_out/pytest_full.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_full.log
