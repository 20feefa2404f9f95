"""Kernel timeline of one vrb_build (CUPTI through torch.profiler): every
kernel / memcpy / memset on the device with its start and duration, and the
idle gaps between them, to find host-side stalls inside a build.
usage: python tools/timeline.py C5B [min_gap_us]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1809_04424_b200 as vrb  # noqa: E402
import workloads  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5B"
min_gap = float(sys.argv[2]) if len(sys.argv) > 2 else 15.0
w = workloads.WORKLOADS[cfg]
X = torch.from_numpy(w.points()).cuda()
vrb.use_torch_allocator(True)
for _ in range(3):
    r = vrb.build(X, maxdim=w.maxdim, radius=w.radius)
    torch.cuda.synchronize()
    del r
with profile(activities=[ProfilerActivity.CPU, ProfilerActivity.CUDA]) as prof:
    r = vrb.build(X, maxdim=w.maxdim, radius=w.radius)
    torch.cuda.synchronize()
dev, host = [], []
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        dev.append((e.time_range.start, e.time_range.end, e.name))
    else:
        host.append((e.time_range.start, e.time_range.end, e.name))
dev.sort()
host.sort()
t0 = dev[0][0]
busy = sum(b - a for a, b, _ in dev)
span = dev[-1][1] - t0
print(f"{cfg}: {len(dev)} device ops, span {span / 1e3:.3f} ms, busy {busy / 1e3:.3f} ms, "
      f"idle {(span - busy) / 1e3:.3f} ms")
prev_end, prev_name = dev[0][1], dev[0][2]
gaps = []
for a, b, nm in dev[1:]:
    if a - prev_end > min_gap:
        # host calls overlapping the gap
        hc = [h[2] for h in host if h[0] < a and h[1] > prev_end and "cuda" in h[2].lower()]
        gaps.append((a - prev_end, prev_name[:40], nm[:40], sorted(set(hc))[:4]))
    prev_end, prev_name = max(prev_end, b), nm
if os.environ.get("TL_ALL"):
    for a, b, nm in dev:
        print(f"{(a - t0) / 1e3:9.3f} ms {(b - a):9.1f} us  {nm[:90]}")
for g, p, q, hc in gaps:
    print(f"gap {g:8.1f} us after {p:40s} before {q:40s} {hc}")
print(f"gaps > {min_gap} us: {len(gaps)}, total {sum(g[0] for g in gaps) / 1e3:.3f} ms")
