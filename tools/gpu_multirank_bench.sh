#!/bin/bash
# bench.py under torchrun with N ranks on ONE GPU over gloo (the N > 1 code path of the
# driver's scaling run; timings are not multi-GPU numbers).  usage: bash tools/gpu_multirank_bench.sh tag N W
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=$1; N=${2:-2}; W=${3:-C3}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
VRB_DIST_BACKEND=gloo timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus $N --workload $W --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/${TAG}_mr_${W}_${N}.json 2> gpurun_out/${TAG}_mr_${W}_${N}.err
echo "rc=$?"; tail -c 1500 gpurun_out/${TAG}_mr_${W}_${N}.json; tail -3 gpurun_out/${TAG}_mr_${W}_${N}.err
