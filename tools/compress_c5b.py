"""One build of a workload, then vrb_compress_d2 (F1 clear and compress)
three times, device-timed: the target command for ncu on the compress
kernels.  Usage: python tools/compress_c5b.py [workload]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_04424_b200 as vrb  # noqa: E402
import workloads  # noqa: E402

w = workloads.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "C5B"]
vrb.use_torch_allocator(True)
r = vrb.build(torch.from_numpy(w.points()).cuda(), maxdim=w.maxdim, radius=w.radius)
r.h0()
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    cp, rv, rm = r.compress_d2()
    e1.record()
    torch.cuda.synchronize()
    print("compress ms", round(e0.elapsed_time(e1), 2), "nnz", rv.shape[0], "rows", rm.shape[0], flush=True)
    del cp, rv, rm
r.free()
