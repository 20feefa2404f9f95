"""One (or a few) vrb_build calls of a workload: the target command for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_04424_b200 as vrb  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5B"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
w = workloads.WORKLOADS[cfg]
npts = int(sys.argv[3]) if len(sys.argv) > 3 else None   # optional: first npts points only
P = w.points()
if w.kind == "matrix":
    P = P[:npts, :npts] if npts else P
else:
    P = P[:npts]
X = torch.from_numpy(P.copy()).cuda()
vrb.use_torch_allocator(True)
for _ in range(reps):
    r = (vrb.build_dm(X, maxdim=w.maxdim, radius=w.radius) if w.kind == "matrix"
         else vrb.build(X, maxdim=w.maxdim, radius=w.radius))
    torch.cuda.synchronize()
    print("edge path", vrb.last_edge_path())
    del r
print("done", cfg, reps)
