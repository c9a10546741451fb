"""kgsynth v0 -- seeded synthetic TransE-shaped embeddings.

This module is shared by the oracle side and the CUDA side ONLY as an input
generator: it draws random numbers and nothing else.  It holds none of the
method's arithmetic (no distances, no pivots, no sorting, no thresholds).

Recipe:

* ``cluster`` (primary; relations translate one entity cluster onto another,
  the structure a trained TransE model has -- PAPER.md:193 "h + r ~ t"):
    K   = max(4, round(sqrt(N) / 2))
    u   ~ N(0, I_d)  (K x d), rows normalised
    s   ~ U[0, 1)    (K x 1)
    C   = u * s * sqrt(d)                      cluster centres, norms in [0, sqrt d)
    lab ~ U{0..K-1}  (N)
    E   = C[lab] + 0.05 * N(0, I_d)
    a,b ~ U{0..K-1}  (R each)
    Rel = C[b] - C[a] + 0.02 * N(0, I_d)
* ``uniform`` (control: almost nothing prunes):
    E ~ U[-1, 1)^{N x d},  Rel ~ 0.1 * U[-1, 1)^{R x d}
  (per-dimension range ~2, like the FB15K range 1.9864 quoted at PAPER.md:128).

Draws use numpy's PCG64 ``default_rng(seed)`` in float64 and are cast to
float32, so the same seed gives bit-identical inputs on every machine.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

GENERATOR_VERSION = "kgsynth-v0"


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    N: int
    R: int
    d: int
    seed: int
    dist: str = "cluster"
    note: str = ""


# BASELINE.json "configs", in order.  Seeds C1..C5 = 1..5.
CONFIGS = {
    "c1": Config("c1", 1000, 10, 50, 1, note="TransE L2 tiny, ~0.1% hits (CPU brute force in seconds)"),
    "c2": Config("c2", 40943, 18, 100, 2, note="WN18-shaped, L1 and L2"),
    "c3": Config("c3", 14951, 1345, 100, 3, note="FB15k-shaped, L2, hit-rate sweep 1e-6..1e-3"),
    "c4": Config("c4", 123182, 37, 200, 4, note="YAGO3-10-shaped, L2"),
    "c5": Config("c5", 1000000, 100, 128, 5, note="synthetic 1M entities, L2"),
}


def generate(N: int, R: int, d: int, seed: int, dist: str = "cluster"):
    """Return (E, Rel) as C-contiguous float32 arrays of shape (N, d), (R, d)."""
    rng = np.random.default_rng(seed)
    if dist == "cluster":
        K = max(4, int(round(math.sqrt(N) / 2)))
        u = rng.standard_normal((K, d))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        s = rng.random((K, 1))
        C = u * s * math.sqrt(d)
        lab = rng.integers(0, K, size=N)
        E = C[lab] + 0.05 * rng.standard_normal((N, d))
        a = rng.integers(0, K, size=R)
        b = rng.integers(0, K, size=R)
        Rel = C[b] - C[a] + 0.02 * rng.standard_normal((R, d))
    elif dist == "uniform":
        E = rng.uniform(-1.0, 1.0, size=(N, d))
        Rel = 0.1 * rng.uniform(-1.0, 1.0, size=(R, d))
    else:
        raise ValueError(f"unknown distribution {dist!r}")
    return (np.ascontiguousarray(E, dtype=np.float32),
            np.ascontiguousarray(Rel, dtype=np.float32))


def generate_se(N: int, R: int, d: int, seed: int, dist: str = "cluster"):
    """SE-shaped inputs (Structured Embedding): entities as ``generate``;
    per relation two d x d matrices W = I + 0.1 / sqrt(d) * N(0, 1) (lhs, rhs), so
    W_lhs h and W_rhs t stay close for nearby entities.  Random draws only."""
    E, _ = generate(N, R, d, seed, dist)
    rng = np.random.default_rng(seed + 7919)
    eye = np.eye(d)
    Wl = (eye + 0.1 / math.sqrt(d) * rng.standard_normal((R, d, d))).astype(np.float32)
    Wr = (eye + 0.1 / math.sqrt(d) * rng.standard_normal((R, d, d))).astype(np.float32)
    return E, Wl, Wr


def generate_config(name: str, dist: str | None = None):
    c = CONFIGS[name]
    return generate(c.N, c.R, c.d, c.seed, dist or c.dist)


def sample_rows(N: int, R: int, S: int, seed: int) -> np.ndarray:
    """Seeded sample of S distinct query rows (row = h * R + r), sorted."""
    rng = np.random.default_rng(10_000 + seed)
    total = N * R
    S = min(S, total)
    if S == total:
        return np.arange(total, dtype=np.int64)
    rows = rng.choice(total, size=S, replace=False)
    return np.sort(rows.astype(np.int64))
