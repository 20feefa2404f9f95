#!/bin/bash
# ncu --set full of the rr count + fill (C5B) and the clear-and-compress column passes
cd "${GRAFT_REPO_ROOT:-/root/repo}"
TAG=${1:-rrp}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1 || exit 1
export VRB_TRI_PATH=rr
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_triangles|k_tri_fill_rr" -s 2 -c 2 -o gpurun_out/${TAG}_tri python tools/one_build.py C5B 2 > gpurun_out/${TAG}_tri.log 2>&1
echo "tri rc=$?"
{ python tools/ncu_summary.py gpurun_out/${TAG}_tri.ncu-rep "" 10; python tools/ncu_lines.py gpurun_out/${TAG}_tri.ncu-rep "k_tri_fill_rr" 25; python tools/ncu_lines.py gpurun_out/${TAG}_tri.ncu-rep "k_triangles" 25; } > gpurun_out/${TAG}_ncu_tri_c5b.txt 2>&1
unset VRB_TRI_PATH
cat > /tmp/cc.py <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_1809_04424_b200 as vrb, workloads
X = torch.from_numpy(workloads.WORKLOADS["C5B"].points()).cuda()
vrb.use_torch_allocator(True)
r = vrb.build(X, maxdim=1, radius=2.8); r.h0(); torch.cuda.synchronize()
cp, rv, rm = r.compress_d2(); torch.cuda.synchronize(); print("ok")
PY
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_col_tile -c 2 -o gpurun_out/${TAG}_cc python /tmp/cc.py > gpurun_out/${TAG}_cc.log 2>&1
echo "cc rc=$?"
{ python tools/ncu_summary.py gpurun_out/${TAG}_cc.ncu-rep "" 10; python tools/ncu_lines.py gpurun_out/${TAG}_cc.ncu-rep "k_col_tile_fill" 20; } > gpurun_out/${TAG}_ncu_cc.txt 2>&1
ls -la gpurun_out/${TAG}_*
