"""Device timing of vrb_gf2_blockprodsum on a synthetic
Schur-block workload: D 2e6 x 1e6 (<= 4 nnz/col), C 2e6 x 1e6 (<= 5 nnz/col),
E 1e6 x 1e6 (<= 4 nnz/col).  Prints one JSON line (ms per call, candidates/s,
output nnz/s).  The paper's blockprodsum numbers (Table `workers`, P:1126-1139:
15.5 s on 1 worker -> 8.3 s on 12, Dragon2) are for Eirene's own blocks:
context only."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1809_04424_b200 as vrb  # noqa: E402
from test_gf2_gpu import dev, rand_csc_fast  # noqa: E402

rng = np.random.default_rng(7)
nr, k, nc = 2_000_000, 1_000_000, 1_000_000
D, C, E = rand_csc_fast(rng, nr, nc, 4), rand_csc_fast(rng, nr, k, 5), rand_csc_fast(rng, k, nc, 4)
Dd, Cd, Ed = dev(D), dev(C), dev(E)
vrb.use_torch_allocator(True)
for _ in range(3):
    S = vrb.gf2_blockprodsum(nr, Dd, Cd, Ed)
    del S
torch.cuda.synchronize()
reps, ms = 5, []
for _ in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    S = vrb.gf2_blockprodsum(nr, Dd, Cd, Ed)
    e1.record()
    torch.cuda.synchronize()
    ms.append(e0.elapsed_time(e1))
    nnz = S.nnz
    del S
ccnt = np.diff(C[0])
cand = int(np.diff(D[0]).sum() + ccnt[E[1].astype(np.int64)].sum())
t = float(np.median(ms))
print(json.dumps({"workload": "F4 blockprodsum synthetic", "nrows": nr, "k": k, "ncols": nc,
                  "nnz_D": int(D[0][-1]), "nnz_C": int(C[0][-1]), "nnz_E": int(E[0][-1]),
                  "candidates": cand, "nnz_S": int(nnz), "ms_median": t, "ms_all": ms,
                  "candidates_per_s": cand / (t / 1e3), "nnz_S_per_s": nnz / (t / 1e3)}))
