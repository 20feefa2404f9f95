"""Per-build stage times of a workload (library CUDA events), one line per build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_04424_b200 as vrb  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5B"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
w = workloads.WORKLOADS[cfg]
X = torch.from_numpy(w.points()).cuda()
vrb.use_torch_allocator(True)
vrb.set_profiling(True)
for i in range(reps):
    r = vrb.build(X, maxdim=w.maxdim, radius=w.radius)
    torch.cuda.synchronize()
    print(cfg, i, {k: round(v, 2) for k, v in vrb.last_stage_ms().items() if v})
    del r
