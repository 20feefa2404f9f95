"""Experiment: does processing hosts in a spatially local order (points
permuted into k-d tree order before the build) cut the C5B fill's gather
traffic?  Times the build stages of C5B as given and permuted."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_04424_b200 as vrb  # noqa: E402
import workloads  # noqa: E402


def kd_order(P, leaf=32):
    idx = np.arange(P.shape[0])
    out = []
    stack = [idx]
    while stack:
        ix = stack.pop()
        if len(ix) <= leaf:
            out.append(ix)
            continue
        sub = P[ix]
        c = int(np.argmax(sub.max(0) - sub.min(0)))
        o = np.argsort(sub[:, c], kind="stable")
        h = len(ix) // 2
        stack.append(ix[o[h:]])
        stack.append(ix[o[:h]])
    return np.concatenate(out)


w = workloads.WORKLOADS["C5B"]
P = w.points()
orders = {"given": np.arange(P.shape[0]), "coord0": np.argsort(P[:, 0], kind="stable"), "kd": kd_order(P)}
vrb.set_profiling(True)
for name, o in orders.items():
    X = torch.from_numpy(np.ascontiguousarray(P[o])).cuda()
    ts = []
    for rep in range(4):
        r = vrb.build(X, maxdim=1, radius=w.radius)
        torch.cuda.synchronize()
        st = vrb.last_stage_ms()
        if rep:
            ts.append(st)
        del r
    print(name, {k: round(float(np.mean([t[k] for t in ts])), 2) for k in ("count", "fill", "total")}, flush=True)
