"""Write tests/golden/<config>_levels.json: oracle-computed digests of the
full-size configs, for the full-size GPU parity tests.

Calls only oracle/ (and the shared input generators in workloads.py).  The
per-level simplex histogram of C3/C5B takes minutes on one core, so it is
stored as a SHA-256 digest plus coarse bucket sums instead of being recomputed
on every GPU test run.

    python tools/make_golden.py C3 C5B C4 HIV
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle      # noqa: E402
import workloads   # noqa: E402

NBUCKETS = 256


def digest(config: str, k: int = 2) -> dict:
    w = workloads.WORKLOADS[config]
    X = w.points()
    t0 = time.time()
    o = oracle.Oracle(None, w.radius, D=X) if w.kind == "matrix" else oracle.Oracle(X, w.radius)
    ev, ef, el, vor = o.edges()
    t1 = time.time()
    hist = o.filt_hist(k)
    t2 = time.time()
    edges = np.concatenate([ev.ravel().astype(np.uint64), ef.astype(np.uint64)])
    buckets = np.array_split(hist, NBUCKETS)
    return {
        "config": config,
        "citation": "computed by tools/make_golden.py with oracle/ only (SURVEY 8(c) steps 1-6); "
                    "hist[f] = number of dim-%d simplices with filt f" % k,
        "points_sha256": hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest(),
        "E": int(o.E),
        "nvals": int(o.nvals),
        "edges_sha256": hashlib.sha256(edges.tobytes()).hexdigest(),
        "value_of_rank_sha256": hashlib.sha256(vor.tobytes()).hexdigest(),
        "dim": k,
        "count": int(hist.sum()),
        "hist_sha256": hashlib.sha256(hist.astype(np.uint64).tobytes()).hexdigest(),
        "hist_bucket_sums": [int(b.sum()) for b in buckets],
        "oracle_seconds": {"edges": round(t1 - t0, 2), "hist": round(t2 - t1, 2)},
    }


def digest_edges(config: str) -> dict:
    # edges only (maxdim 0: C5A's 2e8 edges, full filtration)
    w = workloads.WORKLOADS[config]
    X = w.points()
    t0 = time.time()
    o = oracle.Oracle(X, w.radius)
    ev, ef, el, vor = o.edges()
    t1 = time.time()
    edges = np.concatenate([ev.ravel().astype(np.uint64), ef.astype(np.uint64)])
    return {
        "config": config,
        "citation": "computed by tools/make_golden.py with oracle/ only (SURVEY 8(c) steps 1-4): "
                    "SHA-256 of the oracle's (i, j) pairs and levels in (len, i, j) order, and of value_of_rank",
        "points_sha256": hashlib.sha256(np.ascontiguousarray(X).tobytes()).hexdigest(),
        "E": int(o.E),
        "nvals": int(o.nvals),
        "edges_sha256": hashlib.sha256(edges.tobytes()).hexdigest(),
        "value_of_rank_sha256": hashlib.sha256(vor.tobytes()).hexdigest(),
        "oracle_seconds": {"edges": round(t1 - t0, 2)},
    }


if __name__ == "__main__":
    for cfg in sys.argv[1:] or ["C3", "C5B", "C4"]:
        if workloads.WORKLOADS[cfg].maxdim == 0:
            d = digest_edges(cfg)
            path = os.path.join(ROOT, "tests", "golden", f"{cfg.lower()}_edges.json")
            with open(path, "w") as f:
                json.dump(d, f, indent=1)
            print(cfg, d["E"], d["oracle_seconds"])
            continue
        d = digest(cfg, k=3 if workloads.WORKLOADS[cfg].maxdim >= 2 else 2)
        path = os.path.join(ROOT, "tests", "golden", f"{cfg.lower()}_levels.json")
        with open(path, "w") as f:
            json.dump(d, f, indent=1)
        print(cfg, d["E"], d["count"], d["oracle_seconds"])
