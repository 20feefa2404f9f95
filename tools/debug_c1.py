import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle, workloads, paper_1809_04424_b200 as vrb
w = workloads.WORKLOADS["C1"]; X = w.points()
res = vrb.build(X, maxdim=1, radius=w.radius)
o = oracle.Oracle(X, w.radius)
tv, tf, tr = o.simplices(2)
gtv = res.simplices(2)[0].cpu().numpy().view(np.uint32)
gr = res.boundary(2).cpu().numpy().view(np.uint32)
bad = np.nonzero((gtv != tv).any(1))[0]
print("bad triangles", len(bad), bad[:40])
owners = tr[bad, 2]
print("owner edges", np.unique(owners))
ev = o.edges()[0]
for p in np.unique(owners)[:5]:
    sel = np.nonzero(tr[:, 2] == p)[0]
    print("edge", p, ev[p], "slots", sel[0], sel[-1], "n", len(sel))
    for q in sel:
        print("   ", q, tv[q], gtv[q], tr[q], gr[q], "BAD" if q in bad else "")
