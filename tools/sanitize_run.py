"""Small builds through every entry point, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck): python tools/sanitize_run.py"""
import math
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1809_04424_b200 as vrb  # noqa: E402
import workloads  # noqa: E402

torch.cuda.set_device(0)
for seed, (n, d, kind, r, md) in enumerate([(50, 3, "uniform", math.inf, 2), (120, 3, "lattice", 1.5, 2),
                                           (200, 4, "gauss", 1.2, 1), (90, 2, "dups", 0.3, 2), (3, 3, "uniform", 1.0, 2),
                                           (120, 3, "uniform", math.inf, 2)]):   # apex runs > 104
    X = workloads.random_cloud(seed, n, d, kind)
    res = vrb.build(X, maxdim=md, radius=r)
    res.h0()
    for k in range(1, md + 2):
        res.simplices(k)
        res.boundary_colptr(k)
    del res
w = workloads.WORKLOADS["C2"]
res = vrb.build(w.points()[:400], maxdim=2, radius=w.radius)
res.h0()
del res
D = np.abs(np.subtract.outer(np.arange(60.0), np.arange(60.0))) % 7
vrb.build_dm(D, maxdim=2, radius=3.0)
# round 2 paths: rowsare="dimensions", clear-and-compress, an owner edge with
# > 512 triangles (k_tets_big, dense and sparse), the HIV-like tie sort (keys
# only, rows from the position table)
X = workloads.random_cloud(7, 150, 3, "gauss")
r2 = vrb.build(np.ascontiguousarray(X.T), maxdim=2, radius=1.0, rowsare="dimensions")
r2.compress_d2()
del r2
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_limits_gpu import big_apex_matrix  # noqa: E402
for sparse in ("0", "1"):
    os.environ["VRB_FORCE_SPARSE_TETS"] = sparse
    for tie in (False, True):
        vrb.build_dm(big_apex_matrix(m_apex=600, clique=10, tie=tie), maxdim=2, radius=1.0)
os.environ.pop("VRB_FORCE_SPARSE_TETS")
H = workloads.hamming_matrix(workloads.hamming_sequences(3, n=140, length=120, clades=4))
vrb.build_dm(H, maxdim=1, radius=math.inf)
vrb.build_dm(H, maxdim=2, radius=60.0)
# round 2, second session: the x-major triangle path; the fused edge
# epilogue over several tiles with runs of equal high bits (tied and
# distinct lengths) and a fallback run longer than 64
os.environ["VRB_TRI_PATH"] = "xmajor"
vrb.build(workloads.random_cloud(11, 300, 4, "gauss"), maxdim=1, radius=1.8)
os.environ.pop("VRB_TRI_PATH")
for m in (50, 150):
    theta = np.linspace(0.0, 2.0 * np.pi, m, endpoint=False)
    rad = 1.0 + np.arange(m)[::-1] * 1e-12
    ring = np.stack([rad * np.cos(theta), rad * np.sin(theta)], axis=1)
    vrb.build(np.concatenate([np.zeros((1, 2)), ring, ring[::-1], [[1000.0, 0.0]]]), maxdim=1, radius=math.inf)
vrb.latlon2euc(torch.rand(100, 2, dtype=torch.float64, device="cuda") * 90)
vrb.sortperm_f64(torch.randn(5000, dtype=torch.float64, device="cuda"))
cp = torch.tensor([0, 2, 3], dtype=torch.int64, device="cuda")
rv = torch.tensor([0, 1, 1], dtype=torch.int32, device="cuda")
vrb.gf2_blockprodsum(2, (cp, rv), (cp, rv), (cp, rv))
torch.cuda.synchronize()
print("sanitize run ok")
# round 2, third session: the S3 bucket path (several chunks, refinement,
# sliced scatter) and the forced radix path on the same cloud
Xb = workloads.random_cloud(11, 2500, 10, "gauss")
vrb.build(Xb, maxdim=0, radius=math.inf)
vrb.build(Xb, maxdim=1, radius=2.0)
os.environ["VRB_BK_PASSES"] = "3"
vrb.build(Xb, maxdim=0, radius=math.inf)
del os.environ["VRB_BK_PASSES"]
os.environ["VRB_EDGE_PATH"] = "radix"
vrb.build(Xb, maxdim=0, radius=math.inf)
del os.environ["VRB_EDGE_PATH"]
torch.cuda.synchronize()
print("sanitize_run done")

