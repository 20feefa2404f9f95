"""Randomised parity sweep (GPU vs oracle, element by element): many seeded
small clouds of every kind, capped and full, maxdim 0..2, both S3 paths.
Usage: python tools/stress_parity.py [count]"""
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402,F401

import paper_1809_04424_b200 as vrb  # noqa: E402
import workloads  # noqa: E402
from test_parity_gpu import compare  # noqa: E402

count = int(sys.argv[1]) if len(sys.argv) > 1 else 300
fails = 0
for seed in range(count):
    rng = np.random.default_rng(90000 + seed)
    kind = ["uniform", "gauss", "lattice", "halfint", "dups"][seed % 5]
    n = int(rng.integers(0, 90))
    d = int(rng.integers(1, 7))
    X = workloads.random_cloud(90000 + seed, n, d, kind) * float(10.0 ** rng.integers(-3, 4))
    radius = float(rng.choice([math.inf, 0.3, 0.8, 1.5, 3.0])) * (1.0 if kind in ("lattice", "halfint") else 1.0)
    maxdim = int(rng.integers(0, 3))
    os.environ["VRB_EDGE_PATH"] = ["bucket", "radix"][seed % 2]
    try:
        compare(vrb, X, maxdim, radius, strict=bool(seed % 7 == 3))
    except AssertionError as e:
        fails += 1
        print("FAIL seed", seed, kind, n, d, radius, maxdim, os.environ["VRB_EDGE_PATH"], str(e)[:200], flush=True)
print("stress done", count, "cases,", fails, "failures")
