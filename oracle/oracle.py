"""oracle.py -- TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

CPU definitions of what the hot path computes, written from PAPER.md and
nothing else.  Each function cites the passage it follows (P:NNN = PAPER.md
line NNN).  Nothing here is imported by the product package; the product path
never calls it.

Pins (tests/test_oracle_*.py) tie every function to something other than
itself: hand-worked examples, closed forms, scipy's cdist, brute force,
invariants.  ``pivot_distances`` and ``compute_range`` are pinned the same way.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
_SRC = _HERE / "kgc_oracle.c"
_LIB = _HERE / "libkgc_oracle.so"

TRIPLET_DTYPE = np.dtype([("h", np.int32), ("r", np.int32), ("t", np.int32),
                          ("pad", np.int32), ("dist", np.float64)])


class _Triplet(ctypes.Structure):
    _fields_ = [("h", ctypes.c_int32), ("r", ctypes.c_int32), ("t", ctypes.c_int32),
                ("pad", ctypes.c_int32), ("dist", ctypes.c_double)]


def build(force: bool = False) -> Path:
    """Compile the plain-C oracle (gcc, -O2, no fast-math => index-order FP64 sums)."""
    if force or not _LIB.exists() or _LIB.stat().st_mtime < _SRC.stat().st_mtime:
        tmp = _LIB.with_suffix(f".so.tmp{os.getpid()}")
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", str(tmp), str(_SRC), "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(_LIB))
        L.kgco_dist3.restype = ctypes.c_double
        L.kgco_dist3.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int32] * 2
        L.kgco_dist_rows.restype = ctypes.c_int32
        L.kgco_dist_rows.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                     ctypes.c_int32, ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
                                     ctypes.c_void_p, ctypes.c_int32]
        L.kgco_join.restype = ctypes.c_int64
        L.kgco_join.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                ctypes.c_int32, ctypes.c_int32, ctypes.c_double, ctypes.c_void_p,
                                ctypes.c_int64, ctypes.c_int32, ctypes.POINTER(ctypes.POINTER(_Triplet))]
        L.kgco_free.argtypes = [ctypes.c_void_p]
        L.kgco_threads_used.restype = ctypes.c_int32
        _lib = L
    return _lib


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


# --------------------------------------------------------------------------
# dist3 and the join (Definition 1; TransE; Fig. naive)
# --------------------------------------------------------------------------

def dist3(h, r, t, norm: int) -> float:
    """dist3(h, r, t) = ||h + r - t||_{L_p}, FP64, index-order sum."""
    h, r, t = _f32(h), _f32(r), _f32(t)
    return lib().kgco_dist3(h.ctypes.data, r.ctypes.data, t.ctypes.data, h.shape[0], norm)


def dist_rows(E, Rel, norm: int, rows=None, threads: int = 0) -> np.ndarray:
    """FP64 dist3 of query rows (row = h*R + r) against every tail: (len(rows), N)."""
    E, Rel = _f32(E), _f32(Rel)
    N, d = E.shape
    R = Rel.shape[0]
    rows_arr = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    n = N * R if rows_arr is None else rows_arr.shape[0]
    out = np.empty((n, N), dtype=np.float64)
    rc = lib().kgco_dist_rows(E.ctypes.data, Rel.ctypes.data, N, R, d, norm,
                              None if rows_arr is None else rows_arr.ctypes.data, n,
                              out.ctypes.data, threads)
    if rc != 0:
        raise ValueError("kgco_dist_rows failed")
    return out


def join(E, Rel, norm: int, eps: float, rows=None, threads: int = 0) -> np.ndarray:
    """All (h, r, t) with dist3 <= eps (Definition 1), as a TRIPLET_DTYPE array
    ordered by (h, r, t) (or by the given row order, then t)."""
    E, Rel = _f32(E), _f32(Rel)
    N, d = E.shape
    R = Rel.shape[0]
    rows_arr = None if rows is None else np.ascontiguousarray(rows, dtype=np.int64)
    n = 0 if rows_arr is None else rows_arr.shape[0]
    ptr = ctypes.POINTER(_Triplet)()
    cnt = lib().kgco_join(E.ctypes.data, Rel.ctypes.data, N, R, d, norm, float(eps),
                          None if rows_arr is None else rows_arr.ctypes.data, n, threads,
                          ctypes.byref(ptr))
    if cnt < 0:
        raise ValueError(f"kgco_join failed ({cnt})")
    out = np.empty(cnt, dtype=TRIPLET_DTYPE)
    if cnt:
        ctypes.memmove(out.ctypes.data, ptr, cnt * TRIPLET_DTYPE.itemsize)
    lib().kgco_free(ptr)
    return out


def topk(E, Rel, norm: int, k: int, exclude_self: bool = False, threads: int = 0) -> np.ndarray:
    """The k smallest dist3 over all N*R*N triplets (ties broken by (h, r, t)), as a
    TRIPLET_DTYPE array in ascending order -- the paper's minimum-distance statistic
    "min_{i,j,k} ||h_i + r_j - t_k||" (reading R16), with or without self edges
    h = t (P:128 reports both).  Brute force: every distance from ``dist_rows`` (FP64,
    index-order sums), one stable sort.  Small inputs only (N*R*N values in memory)."""
    E, Rel = _f32(E), _f32(Rel)
    N, R = E.shape[0], Rel.shape[0]
    D = dist_rows(E, Rel, norm, threads=threads)            # (N*R, N), row = h*R + r
    h = np.repeat(np.arange(N), R * N)
    r = np.tile(np.repeat(np.arange(R), N), N)
    t = np.tile(np.arange(N), N * R)
    dist = D.ravel()
    keep = h != t if exclude_self else np.ones(dist.size, bool)
    h, r, t, dist = h[keep], r[keep], t[keep], dist[keep]
    order = np.lexsort((t, r, h, dist))[:k]                 # primary key: dist
    out = np.zeros(order.size, dtype=TRIPLET_DTYPE)
    out["h"], out["r"], out["t"], out["dist"] = h[order], r[order], t[order], dist[order]
    return out


def se_connectors(E, Wl, Wr):
    """SE connectors: a_{r,h} = W_r^lhs h and b_{r,t} = W_r^rhs t in FP64,
    shape (R, N, d) each (numpy matmul of the float32 inputs promoted to float64)."""
    E64 = np.asarray(E, np.float64)
    A = np.einsum("rkj,nj->rnk", np.asarray(Wl, np.float64), E64)
    B = np.einsum("rkj,nj->rnk", np.asarray(Wr, np.float64), E64)
    return A, B


def se_join(E, Wl, Wr, eps: float) -> np.ndarray:
    """All (h, r, t) with ||W_r^lhs h - W_r^rhs t||_1 <= eps (SE, Definition 1
    P:92-94), FP64, as TRIPLET_DTYPE ordered by (h, r, t).  Brute force, small inputs."""
    A, B = se_connectors(E, Wl, Wr)
    R, N, _ = A.shape
    rows = []
    for r in range(R):
        D = np.abs(A[r][:, None, :] - B[r][None, :, :]).sum(axis=2)   # (h, t)
        h, t = np.nonzero(D <= eps)
        for hh, tt in zip(h, t):
            rows.append((hh, r, tt, D[hh, tt]))
    rows.sort()
    out = np.zeros(len(rows), dtype=TRIPLET_DTYPE)
    if rows:
        arr = np.array(rows, dtype=np.float64)
        out["h"], out["r"], out["t"], out["dist"] = arr[:, 0], arr[:, 1], arr[:, 2], arr[:, 3]
    return out


def threads_used() -> int:
    return int(lib().kgco_threads_used())


def triplet_count(N: int, R: int) -> int:
    """Number of candidate triplets |E| x |R| x |E| (14,951 x 2,690 x 14,951)."""
    return N * R * N


# --------------------------------------------------------------------------
# Preprocessing of the fast completion algorithm (Fig. algo1 lines 3-11)
# --------------------------------------------------------------------------

def connector1(h, r):
    """TransE connector_1(a, b) = a + b, FP64."""
    return np.asarray(h, np.float64) + np.asarray(r, np.float64)


def connector2(t, r):
    """TransE connector_2(a, b) = a."""
    return np.asarray(t, np.float64)


def pivot_distances(X, pivot, norm: int) -> np.ndarray:
    """Dist(p, Y): ||x - p||_p for every row x, FP64."""
    D = np.asarray(X, np.float64) - np.asarray(pivot, np.float64)[None, :]
    if norm == 1:
        return np.abs(D).sum(axis=1)
    return np.sqrt((D * D).sum(axis=1))


def sort_side(dist_list):
    """Sort distA / distB and rearrange (P:154, P:360 lines 7-10).
    Returns (perm, sorted).  Stable: ties keep ascending original index."""
    dist_list = np.asarray(dist_list)
    perm = np.argsort(dist_list, kind="stable")
    return perm, dist_list[perm]


def compute_range(sa, sb, eps):
    """compute_range of Fig. algo2, reconstructed from its prose.

    s-part (lines 1-14): alternate the i-pointer movement (while
    sb[j] >= sa[i] - eps: s[i] = j, i += 1) and the j-pointer movement (while
    sb[j] < sa[i] - eps: j += 1) until i or j reaches the end; leftover i get
    s[i] = Nj - 1 (lines 12-14).
    e-part (lines 15-27): j-pointer movement (while sb[j] <= sa[i] + eps:
    j += 1), then i-pointer movement e[i] = max(0, j - 1).
    Empty intervals get the paper's "programming convenience" values:
    a one-element range at 0 or Nj - 1 whose candidate verification rejects.
    """
    sa = np.asarray(sa, np.float64)
    sb = np.asarray(sb, np.float64)
    if eps < 0:
        raise ValueError("eps must be >= 0")
    Ni, Nj = len(sa), len(sb)
    s = np.zeros(Ni, dtype=np.int64)
    e = np.zeros(Ni, dtype=np.int64)
    i = j = 0
    while i < Ni and j < Nj:
        while i < Ni and sb[j] >= sa[i] - eps:      # i-pointer movement (line 6)
            s[i] = j
            i += 1
        while i < Ni and j < Nj and sb[j] < sa[i] - eps:   # j-pointer movement (lines 9-10)
            j += 1
    while i < Ni:                                   # lines 12-14
        s[i] = Nj - 1
        i += 1
    i = j = 0
    while i < Ni:
        while j < Nj and sb[j] <= sa[i] + eps:      # j-pointer movement (lines 17-18)
            j += 1
        e[i] = max(0, j - 1)                        # i-pointer movement (lines 20-22)
        i += 1
    return s, e


def ranges_definition(sa, sb, eps):
    """Eq. (11) read literally: s_i / e_i = min / max of
    {j : |sa[i] - sb[j]| <= eps}; an empty set gives s_i > e_i (s=Nj, e=-1).
    O(m n) brute force -- the declarative reference for compute_range."""
    sa = np.asarray(sa, np.float64)
    sb = np.asarray(sb, np.float64)
    m, n = len(sa), len(sb)
    s = np.full(m, n, dtype=np.int64)
    e = np.full(m, -1, dtype=np.int64)
    for i in range(m):
        ok = np.nonzero(np.abs(sa[i] - sb) <= eps)[0]
        if ok.size:
            s[i], e[i] = ok[0], ok[-1]
    return s, e


def group_candidates(s, e, max_group_size: int):
    """Grouping of Fig. algo3: grow [start, i) while
    (e[i-1] - s[start] + 1) * (i - start) <= MAX_GROUP_SIZE; by Lemma 2's
    monotonicity range_min = s[start], range_max = e[i-1].  A single
    over-budget row forms its own group.  Returns (start, cnt, range_min, range_max)."""
    m = len(s)
    groups = []
    start = 0
    while start < m:
        i = start + 1
        while i < m and (e[i] - s[start] + 1) * (i + 1 - start) <= max_group_size:
            i += 1
        groups.append((start, i - start, int(s[start]), int(e[i - 1])))
        start = i
    return groups


# --------------------------------------------------------------------------
# Threshold calibration (reading R14)
# --------------------------------------------------------------------------

def calibrate_theta(E, Rel, norm: int, hit_rate: float, rows, rel_norms_guard: bool = True,
                    tie_guard_rel: float = 2e-4, threads: int = 0):
    """theta at the requested hit rate over the sampled rows (FP64 dist3): the
    midpoint of the k-th and (k+1)-th smallest sampled distances, k = round(hit
    rate x sample size), moved below any self-edge distance ||r_j||_p closer
    than ``tie_guard_rel * theta`` (N-fold ties, reading R14), then rounded to
    float32.  Returns (theta_f32, info)."""
    D = dist_rows(E, Rel, norm, rows, threads).ravel()
    k = min(max(1, int(round(hit_rate * D.size))), D.size - 1) if D.size > 1 else 1
    D.sort()
    theta = 0.5 * (D[k - 1] + D[k]) if D.size > 1 else float(D[0])
    if rel_norms_guard:
        Rel64 = np.asarray(Rel, np.float64)
        guard = np.abs(Rel64).sum(1) if norm == 1 else np.sqrt((Rel64 ** 2).sum(1))
        for _ in range(100):
            close = np.abs(guard - theta) <= tie_guard_rel * theta
            if not close.any():
                break
            theta = float(guard[close].min()) * (1.0 - 2.0 * tie_guard_rel)
    theta = float(np.float32(theta))
    n_hits = int(np.searchsorted(D, theta, side="right"))
    return theta, {"k": k, "sample_hits": n_hits, "sample_pairs": int(D.size),
                   "hit_rate_sample": n_hits / D.size}


# --------------------------------------------------------------------------
# Comparator (BASELINE.json north_star tolerances)
# --------------------------------------------------------------------------

def compare(gpu, orc_loose, eps: float, band_rel: float = 1e-4, dist_rel: float = 1e-5):
    """gpu: array with fields h, r, t, dist.  orc_loose: oracle join run at
    eps * (1 + band_rel).  Checks tight <= gpu <= loose, no duplicates, and
    |d_gpu - d_orc| <= dist_rel * max(d_orc, eps).  Returns a dict of findings."""
    key = lambda a: (a["h"].astype(np.int64) << 42) | (a["r"].astype(np.int64) << 21) | a["t"].astype(np.int64)
    kg = key(gpu)
    ko = key(orc_loose)
    res = {"gpu": int(kg.size), "loose": int(ko.size)}
    ug = np.unique(kg)
    res["duplicates"] = int(kg.size - ug.size)
    tight_mask = orc_loose["dist"] < eps * (1.0 - band_rel)
    kt = ko[tight_mask]
    res["tight"] = int(kt.size)
    res["missing"] = int(np.setdiff1d(kt, ug, assume_unique=False).size)
    res["extra"] = int(np.setdiff1d(ug, ko, assume_unique=False).size)
    order_o = np.argsort(ko)
    pos = np.searchsorted(ko[order_o], kg)
    pos = np.clip(pos, 0, max(0, ko.size - 1))
    match = (ko.size > 0) & (ko[order_o][pos] == kg) if ko.size else np.zeros(kg.size, bool)
    if np.any(match):
        dg = gpu["dist"][match].astype(np.float64)
        do = orc_loose["dist"][order_o][pos][match]
        err = np.abs(dg - do) / np.maximum(do, eps)
        res["max_dist_rel_err"] = float(err.max())
    else:
        res["max_dist_rel_err"] = 0.0
    res["ok"] = (res["duplicates"] == 0 and res["missing"] == 0 and res["extra"] == 0
                 and res["max_dist_rel_err"] <= dist_rel)
    return res
