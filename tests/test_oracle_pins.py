"""Pins for oracle/ (no GPU).  Each test ties the oracle to something other than
itself: a hand-worked / paper-printed value, an independent library routine,
a brute force written differently, or an invariant of the mathematics.
"""
import itertools
import math

import numpy as np
import pytest

from synth import generate


def _keyset(a):
    return set(zip(a["h"].tolist(), a["r"].tolist(), a["t"].tolist()))


# ---- hand-worked values (tests/golden/spec_examples.json, each cited) ----

def test_dist_hand_examples(orc, golden):
    for ex in golden["dist"]:
        got = orc.dist3(ex["h"], ex["r"], ex["t"], ex["norm"])
        assert got == pytest.approx(ex["expect"], rel=1e-15, abs=1e-15), ex["cite"]


def test_join_hand_examples(orc, golden):
    for ex in golden["join"]:
        E = np.array(ex["E"], np.float32)
        Rel = np.array(ex["Rel"], np.float32)
        got = orc.join(E, Rel, ex["norm"], ex["eps"])
        assert sorted(_keyset(got)) == sorted(map(tuple, ex["expect"])), ex["cite"]


def test_triplet_count_fb15k(orc, golden):
    for ex in golden["triplet_count"]:
        assert orc.triplet_count(ex["N"], ex["R"]) == ex["expect"], ex["cite"]


# ---- closed forms / special cases ----

def test_eps_infinite_returns_everything(orc):
    E, Rel = generate(13, 3, 5, seed=7)
    got = orc.join(E, Rel, 2, 1e30)
    assert got.size == 13 * 3 * 13
    # and the order is (h, r, t) ascending
    k = got["h"].astype(np.int64) * 10_000 + got["r"] * 100 + got["t"]
    assert np.all(np.diff(k) > 0)


def test_eps_below_minimum_returns_nothing(orc):
    E, Rel = generate(30, 4, 6, seed=8)
    D = orc.dist_rows(E, Rel, 2)
    got = orc.join(E, Rel, 2, float(D.min()) * 0.999)
    assert got.size == 0


def test_planted_exact_translations(orc):
    """Dyadic values: h + r = t holds exactly in fp32 and in FP64, so the
    planted triplets have distance exactly 0."""
    rng = np.random.default_rng(3)
    N, R, d = 40, 5, 16
    E = (rng.integers(-64, 64, size=(N, d)) / 8.0).astype(np.float32)
    Rel = (rng.integers(-64, 64, size=(R, d)) / 8.0).astype(np.float32)
    planted = []
    for r in range(R):
        h, t = 2 * r, 2 * r + 1
        E[t] = E[h] + Rel[r]
        planted.append((h, r, t))
    for norm in (1, 2):
        got = orc.join(E, Rel, norm, 0.0)
        ks = _keyset(got)
        for p in planted:
            assert p in ks
        assert np.all(got["dist"] == 0.0)


def test_r_zero_gives_self_pairs(orc):
    E, _ = generate(50, 1, 8, seed=9, dist="uniform")
    Rel = np.zeros((2, 8), np.float32)
    for norm in (1, 2):
        got = orc.join(E, Rel, norm, 0.0)
        assert _keyset(got) == {(i, r, i) for i in range(50) for r in range(2)}


# ---- independent implementations ----

def test_dist_rows_vs_scipy_cdist(orc):
    from scipy.spatial.distance import cdist
    E, Rel = generate(200, 3, 64, seed=11, dist="uniform")
    rows = np.arange(200 * 3)
    Q = E.astype(np.float64)[rows // 3] + Rel.astype(np.float64)[rows % 3]
    for norm, metric in ((2, "euclidean"), (1, "cityblock")):
        ours = orc.dist_rows(E, Rel, norm)
        ref = cdist(Q, E.astype(np.float64), metric)
        np.testing.assert_allclose(ours, ref, rtol=1e-12, atol=1e-12)


def _python_bruteforce(E, Rel, norm, eps):
    """Pure-Python triple loop with math.fsum (exactly rounded sums) -- a second,
    independently written brute force of Definition 1."""
    out = set()
    N, d = E.shape
    for h, r, t in itertools.product(range(N), range(Rel.shape[0]), range(N)):
        terms = [(float(E[h, k]) + float(Rel[r, k])) - float(E[t, k]) for k in range(d)]
        if norm == 1:
            dist = math.fsum(abs(x) for x in terms)
        else:
            dist = math.sqrt(math.fsum(x * x for x in terms))
        if dist <= eps:
            out.add((h, r, t))
    return out


@pytest.mark.parametrize("norm", [1, 2])
def test_join_vs_python_bruteforce(orc, norm):
    E, Rel = generate(24, 3, 7, seed=12)
    D = np.sort(orc.dist_rows(E, Rel, norm).ravel())
    eps = 0.5 * (D[150] + D[151])            # mid-gap threshold: ~150 hits, no ties at eps
    assert _keyset(orc.join(E, Rel, norm, eps)) == _python_bruteforce(E, Rel, norm, eps)


# ---- invariants of the mathematics ----

def _outside_band(orc, E, Rel, norm, eps, band=1e-4):
    lo = orc.join(E, Rel, norm, eps * (1 - band))
    hi = orc.join(E, Rel, norm, eps * (1 + band))
    return _keyset(lo), _keyset(hi)


def test_symmetry_negated_relations(orc):
    """||t - r - h|| = ||h + r - t||: R(E, -Rel) = {(t, r, h) : (h, r, t) in R(E, Rel)}."""
    E, Rel = generate(120, 4, 10, seed=13)
    D = np.sort(orc.dist_rows(E, Rel, 2).ravel())
    eps = float(D[300])
    a = _keyset(orc.join(E, Rel, 2, eps))
    lo, hi = _outside_band(orc, E, -Rel, 2, eps)
    mirrored = {(t, r, h) for (h, r, t) in a}
    assert lo <= mirrored <= hi


def test_translation_invariance(orc):
    E, Rel = generate(120, 4, 10, seed=14)
    D = np.sort(orc.dist_rows(E, Rel, 2).ravel())
    eps = float(D[400])
    a = _keyset(orc.join(E, Rel, 2, eps))
    lo, hi = _outside_band(orc, (E + np.float32(3.25)).astype(np.float32), Rel, 2, eps)
    assert lo <= a <= hi


def test_norm_nesting(orc):
    """||x||_2 <= ||x||_1 <= sqrt(d) ||x||_2."""
    E, Rel = generate(100, 3, 9, seed=15)
    eps = 2.0
    l1 = _keyset(orc.join(E, Rel, 1, eps))
    l2 = _keyset(orc.join(E, Rel, 2, eps))
    l1_wide = _keyset(orc.join(E, Rel, 1, eps * math.sqrt(9) * (1 + 1e-9)))
    assert l1 <= l2 <= l1_wide


def test_monotone_in_eps(orc):
    E, Rel = generate(80, 3, 8, seed=16)
    prev = set()
    for eps in (0.5, 1.0, 1.5, 2.5):
        cur = _keyset(orc.join(E, Rel, 2, eps))
        assert prev <= cur
        prev = cur


def test_permutation_equivariance(orc):
    """Permuting entity rows by sigma permutes results by sigma (index bookkeeping)."""
    E, Rel = generate(90, 3, 8, seed=17)
    sigma = np.random.default_rng(1).permutation(90)
    inv = np.argsort(sigma)
    eps = 1.2
    a = _keyset(orc.join(E, Rel, 2, eps))
    b = _keyset(orc.join(E[sigma], Rel, 2, eps))
    assert {(int(sigma[h]), r, int(sigma[t])) for (h, r, t) in b} == a
    assert {(int(inv[h]), r, int(inv[t])) for (h, r, t) in a} == b


def test_sampled_rows_match_full_join(orc):
    E, Rel = generate(70, 5, 6, seed=18)
    full = orc.join(E, Rel, 2, 1.0)
    rows = np.array([3, 17, 100, 349])
    sub = orc.join(E, Rel, 2, 1.0, rows=rows)
    rowset = set(rows.tolist())
    expect = {k for k in _keyset(full) if k[0] * 5 + k[1] in rowset}
    assert _keyset(sub) == expect


# ------------------------------------------------- top-k (P:128 minimum-distance statistic)
def _topk_python(E, Rel, norm, k, exclude_self):
    """Independent brute force: pure Python loops and math.fsum (not oracle.dist_rows)."""
    import math
    items = []
    for h in range(E.shape[0]):
        for r in range(Rel.shape[0]):
            for t in range(E.shape[0]):
                if exclude_self and h == t:
                    continue
                x = [float(E[h, j]) + float(Rel[r, j]) - float(E[t, j]) for j in range(E.shape[1])]
                d = math.fsum(abs(v) for v in x) if norm == 1 else math.sqrt(math.fsum(v * v for v in x))
                items.append((d, h, r, t))
    items.sort()
    return items[:k]


@pytest.mark.parametrize("norm", [1, 2])
@pytest.mark.parametrize("exclude_self", [False, True])
def test_topk_matches_python_brute_force(orc, norm, exclude_self):
    rng = np.random.default_rng(11 + norm)
    E = rng.standard_normal((9, 4)).astype(np.float32)
    Rel = (0.3 * rng.standard_normal((3, 4))).astype(np.float32)
    got = orc.topk(E, Rel, norm, 25, exclude_self=exclude_self)
    ref = _topk_python(E, Rel, norm, 25, exclude_self)
    assert [(int(a), int(b), int(c)) for a, b, c in zip(got["h"], got["r"], got["t"])] == [x[1:] for x in ref]
    np.testing.assert_allclose(got["dist"], [x[0] for x in ref], rtol=1e-12, atol=1e-12)


def test_topk_planted_translation_and_self_edges(orc):
    """r = 0 makes every self edge a 0-distance hit; a planted exact translation t = h + r
    (dyadic values) is the unique 0 once self edges are excluded."""
    E = np.array([[0, 0], [1, 1], [3, 0], [0.5, 2]], np.float32)
    Rel = np.array([[0, 0], [2, -1]], np.float32)      # E[1] + Rel[1] == E[2] exactly
    top = orc.topk(E, Rel, 2, 6)
    zero = {(int(h), int(r), int(t)) for h, r, t, d in zip(top["h"], top["r"], top["t"], top["dist"]) if d == 0}
    assert zero == {(0, 0, 0), (1, 0, 1), (2, 0, 2), (3, 0, 3), (1, 1, 2)} and top["dist"][5] > 0
    top1 = orc.topk(E, Rel, 2, 1, exclude_self=True)
    assert (int(top1["h"][0]), int(top1["r"][0]), int(top1["t"][0])) == (1, 1, 2) and top1["dist"][0] == 0


def test_topk_prefix_and_join_consistency(orc):
    """top-k is a prefix of top-(k+m); the k-th distance theta_k gives join(theta_k) >= k rows."""
    rng = np.random.default_rng(5)
    E = rng.standard_normal((30, 6)).astype(np.float32)
    Rel = (0.2 * rng.standard_normal((4, 6))).astype(np.float32)
    a, b = orc.topk(E, Rel, 2, 10), orc.topk(E, Rel, 2, 40)
    assert np.array_equal(a, b[:10])
    assert np.all(np.diff(b["dist"]) >= 0)
    j = orc.join(E, Rel, 2, float(b["dist"][-1]) * (1 + 1e-12))
    assert j.size >= 40 and np.all(np.sort(j["dist"])[:40] == b["dist"])


# ------------------------------------------------- SE (Structured Embedding)
def test_se_identity_matrices_reduce_to_entity_l1(orc):
    """W_lhs = W_rhs = I: dist3 = ||h - t||_1 (scipy cityblock, an independent library)."""
    from scipy.spatial.distance import cdist
    rng = np.random.default_rng(2)
    E = rng.standard_normal((40, 7)).astype(np.float32)
    W = np.stack([np.eye(7, dtype=np.float32)] * 2)
    D = cdist(E.astype(np.float64), E.astype(np.float64), "cityblock")
    eps = float(np.sort(D.ravel())[300])
    got = orc.se_join(E, W, W, eps)
    h, t = np.nonzero(D <= eps)
    assert got.size == 2 * h.size
    assert set(zip(got["h"].tolist(), got["t"].tolist())) == set(zip(h.tolist(), t.tolist()))
    np.testing.assert_allclose(got["dist"], D[got["h"], got["t"]], rtol=1e-12, atol=1e-12)


def test_se_matches_python_brute_force(orc):
    import math
    rng = np.random.default_rng(4)
    E = rng.standard_normal((8, 3)).astype(np.float32)
    Wl = rng.standard_normal((2, 3, 3)).astype(np.float32)
    Wr = rng.standard_normal((2, 3, 3)).astype(np.float32)
    ref = []
    for h in range(8):
        for r in range(2):
            a = [math.fsum(float(Wl[r, k, j]) * float(E[h, j]) for j in range(3)) for k in range(3)]
            for t in range(8):
                b = [math.fsum(float(Wr[r, k, j]) * float(E[t, j]) for j in range(3)) for k in range(3)]
                ref.append((math.fsum(abs(x - y) for x, y in zip(a, b)), h, r, t))
    eps = sorted(x[0] for x in ref)[40]
    got = orc.se_join(E, Wl, Wr, eps)
    want = sorted((h, r, t) for d, h, r, t in ref if d <= eps)
    assert [(int(a), int(b), int(c)) for a, b, c in zip(got["h"], got["r"], got["t"])] == want


def test_se_planted_exact_match(orc):
    """W_lhs = 2I, W_rhs = I and E_t = 2 E_h exactly (dyadic) -> distance 0."""
    E = np.array([[0.5, 1.0], [1.0, 2.0], [3.0, -1.0]], np.float32)
    Wl = np.array([2 * np.eye(2)], np.float32)
    Wr = np.array([np.eye(2)], np.float32)
    got = orc.se_join(E, Wl, Wr, 0.0)
    assert {(int(h), int(t)) for h, t in zip(got["h"], got["t"])} == {(0, 1)} and got["dist"][0] == 0
