"""Time the build stages of a workload (CUDA events inside the library)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_04424_b200 as vrb  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5B"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
w = workloads.WORKLOADS[cfg]
X = torch.from_numpy(w.points()).cuda()
vrb.use_torch_allocator(True)
r = vrb.build(X, maxdim=w.maxdim, radius=w.radius)
del r
vrb.set_profiling(True)
acc = {}
for _ in range(reps):
    r = vrb.build(X, maxdim=w.maxdim, radius=w.radius)
    torch.cuda.synchronize()
    for k, v in vrb.last_stage_ms().items():
        acc[k] = acc.get(k, 0.0) + v / reps
    del r
print(cfg, os.environ.get("VRB_DEBUG_FILL", "0"), {k: round(v, 2) for k, v in acc.items()})
