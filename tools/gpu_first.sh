#!/bin/bash
# first GPU session: build, smoke, small parity tests, benches
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -x -q -k "not full_size and not c5a" > gpurun_out/pytest_small.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_small.log
timeout 600 python bench.py --workload C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_c3.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c3.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c5b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_c5b.log
