"""Seeded synthetic point clouds for the Vietoris-Rips filtration build.

This module holds ONLY input generators: it contains none of the method's
arithmetic (no distances, ranks, cliques, sorts or boundaries).  It is the one
module shared by the oracle tests, the GPU parity tests and ``bench.py``; both
sides read the very same float64 bytes.

The workloads are the five ``BASELINE.json`` configs made concrete in
SURVEY.md section 8(d) (table "Configs as concrete synthetic inputs"); the
recipe of each generator is restated in DESIGN.md section "Input recipe".
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np


@dataclasses.dataclass(frozen=True)
class Workload:
    name: str          # C1 .. C5B
    config: str        # the BASELINE.json config string it realises
    maxdim: int        # homology dimension; simplices are built up to K = maxdim + 1
    radius: float      # inclusive cap on edge length (math.inf = full filtration)
    seed: int
    kind: str = "points"   # "points": n x d cloud; "matrix": n x n distance matrix

    def points(self) -> np.ndarray:
        return _GENERATORS[self.name](self.seed)


def _c1(seed: int) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, 1.0, (50, 3))


def torus_grid(p_count: int, q_count: int, R: float = 1.0, a: float = 0.4) -> np.ndarray:
    """Grid on a torus of major radius R and minor radius a, p-major order.
    u_p = 2*pi*p/p_count (minor angle), v_q = 2*pi*q/q_count (major angle)."""
    pts = []
    for p in range(p_count):
        u = 2.0 * math.pi * p / p_count
        for q in range(q_count):
            v = 2.0 * math.pi * q / q_count
            pts.append(((R + a * math.cos(u)) * math.cos(v),
                        (R + a * math.cos(u)) * math.sin(v),
                        a * math.sin(u)))
    return np.asarray(pts, dtype=np.float64)


def circle_points(count: int, center=(3.5, 0.0, 0.0), radius: float = 1.0) -> np.ndarray:
    """Evenly spaced points (cx + r cos t, cy, cz + r sin t), t = 2*pi*s/count."""
    pts = []
    for s in range(count):
        t = 2.0 * math.pi * s / count
        pts.append((center[0] + radius * math.cos(t), center[1], center[2] + radius * math.sin(t)))
    return np.asarray(pts, dtype=np.float64)


def fibonacci_sphere(count: int) -> np.ndarray:
    """s = i + 0.5, phi = arccos(1 - 2 s / count), theta = pi (1 + sqrt 5) s."""
    i = np.arange(count, dtype=np.float64)
    s = i + 0.5
    phi = np.arccos(1.0 - 2.0 * s / count)
    theta = math.pi * (1.0 + math.sqrt(5.0)) * s
    return np.stack([np.cos(theta) * np.sin(phi), np.sin(theta) * np.sin(phi), np.cos(phi)], axis=1)


def _c2(seed: int) -> np.ndarray:
    base = np.concatenate([torus_grid(20, 35), circle_points(300)], axis=0)
    return base + 0.01 * np.random.default_rng(seed).normal(size=base.shape)


def _c3(seed: int) -> np.ndarray:
    return np.random.default_rng(seed).uniform(0.0, 1.0, (2000, 3))


def _c4(seed: int) -> np.ndarray:
    base = fibonacci_sphere(5000)
    return base + 0.005 * np.random.default_rng(seed).normal(size=base.shape)


def _c5(seed: int) -> np.ndarray:
    return np.random.default_rng(seed).standard_normal((20000, 10))


def hamming_sequences(seed: int, n: int = 1088, length: int = 1000, clades: int = 16, p_clade: float = 0.08,
                      p_leaf: float = 0.03) -> np.ndarray:
    """n synthetic genomic sequences over a 4-letter alphabet (uint8, n x
    length): a random root, `clades` ancestors each with a fraction p_clade of
    its sites mutated, and every sequence its clade ancestor (i mod clades)
    with a fraction p_leaf of its sites mutated (a mutation replaces the
    letter by one of the 3 others).  A two-level star phylogeny: the shape of
    the HIV benchmark's input (1088 genomic sequences of the HIV virus,
    P:520-521), whose Hamming distances tie heavily."""
    rng = np.random.default_rng(seed)
    root = rng.integers(0, 4, length)

    def mutate(a, p):
        a = a.copy()
        m = rng.random(length) < p
        a[m] = (a[m] + rng.integers(1, 4, int(m.sum()))) % 4
        return a

    anc = [mutate(root, p_clade) for _ in range(clades)]
    return np.stack([mutate(anc[i % clades], p_leaf) for i in range(n)]).astype(np.uint8)


def hamming_matrix(seqs: np.ndarray) -> np.ndarray:
    """D[i][j] = number of sites where sequences i and j differ (float64; the
    input of the distance-matrix build, not a step of it).  Counted as
    length - (one-hot agreements), exact in float64 for lengths < 2^53."""
    n, length = seqs.shape
    onehot = np.zeros((n, length * 4), dtype=np.float64)
    onehot[np.repeat(np.arange(n), length), (np.arange(length) * 4)[None, :].repeat(n, 0).ravel() + seqs.ravel()] = 1.0
    same = onehot @ onehot.T
    D = length - same
    np.fill_diagonal(D, 0.0)
    return np.ascontiguousarray(D)


def _hiv(seed: int) -> np.ndarray:
    return hamming_matrix(hamming_sequences(seed))


_GENERATORS = {"C1": _c1, "C2": _c2, "C3": _c3, "C4": _c4, "C5A": _c5, "C5B": _c5, "HIV": _hiv}

WORKLOADS = {
    "C1": Workload("C1", "50 uniform random points in R^3, max dim 1 (edges + triangles), full filtration",
                   1, math.inf, 1),
    "C2": Workload("C2", "1,000-point noisy circle + torus mixture in R^3, max dim 2 (tetrahedra), radius-capped",
                   2, 0.45, 2),
    "C3": Workload("C3", "2,000 uniform points in unit cube R^3, max dim 1, full filtration (Eirene benchmark scale)",
                   1, math.inf, 3),
    "C4": Workload("C4", "5,000-point noisy 2-sphere in R^3, max dim 2 with radius threshold, sharded across 8 GPUs",
                   2, 0.40, 4),
    "C5A": Workload("C5A", "20,000 Gaussian points in R^10, distance + edge ranking (max dim 0)",
                    0, math.inf, 5),
    "C5B": Workload("C5B", "20,000 Gaussian points in R^10, max dim 1, distance + edge ranking + triangle build at 1/2/4/8 GPUs",
                    1, 2.8, 5),
    # the paper's tie-heavy benchmark (not a BASELINE.json config): HIV's 1088
    # genomic sequences as a Hamming distance matrix (Table tab1
    # P:1054-1069), the distance-matrix input of F3, max dim 1 (Eirene's
    # default), full filtration
    "HIV": Workload("HIV", "HIV analog: Hamming distance matrix of 1088 synthetic genomic sequences, max dim 1, "
                           "full filtration (P:520-521)", 1, math.inf, 6, "matrix"),
}


# ----------------------------------------------------------------------------
# Small seeded clouds for the parity suites (random shapes, ties, duplicates).
# ----------------------------------------------------------------------------

def random_cloud(seed: int, n: int, d: int, kind: str = "uniform") -> np.ndarray:
    """kind: 'uniform' (U[0,1)), 'gauss' (N(0,1)), 'lattice' (integers 0..3: heavy
    length ties), 'dups' (uniform with ~25% duplicated points), 'halfint'
    (multiples of 0.5: ties plus non-integer squares)."""
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.uniform(0.0, 1.0, (n, d))
    if kind == "gauss":
        return rng.standard_normal((n, d))
    if kind == "lattice":
        return rng.integers(0, 4, (n, d)).astype(np.float64)
    if kind == "halfint":
        return rng.integers(0, 7, (n, d)).astype(np.float64) * 0.5
    if kind == "dups":
        base = rng.uniform(0.0, 1.0, (n, d))
        if n >= 2:
            k = max(1, n // 4)
            src = rng.integers(0, n, k)
            dst = rng.integers(0, n, k)
            base[dst] = base[src]
        return base
    raise ValueError(kind)


def integer_lattice(side: int, d: int) -> np.ndarray:
    """All points of {0..side-1}^d in lexicographic order."""
    grids = np.meshgrid(*([np.arange(side, dtype=np.float64)] * d), indexing="ij")
    return np.stack([g.reshape(-1) for g in grids], axis=1)


def circle_jitter(count: int = 50, jitter: float = 1e-3, seed: int = 0) -> np.ndarray:
    """Evenly spaced unit circle in the plane plus uniform jitter."""
    t = 2.0 * np.pi * np.arange(count) / count
    base = np.stack([np.cos(t), np.sin(t)], axis=1)
    return base + jitter * np.random.default_rng(seed).uniform(-1.0, 1.0, base.shape)
