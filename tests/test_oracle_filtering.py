"""Pins for the oracle's filtering steps: Lemma 1, Lemma 2 /
compute_range (Fig. algo2), grouping."""
import numpy as np
import pytest

from synth import generate


def test_compute_range_spec_example(orc, golden):
    for ex in golden["compute_range"]:
        s, e = orc.compute_range(ex["sa"], ex["sb"], ex["eps"])
        assert s.tolist() == ex["s"] and e.tolist() == ex["e"], ex["cite"]


def test_compute_range_all_pass_and_disjoint(orc):
    s, e = orc.compute_range([1.0, 2.0], [0.0, 5.0, 9.0], 100.0)
    assert s.tolist() == [0, 0] and e.tolist() == [2, 2]
    # disjoint: the paper's convenience range is one index whose check fails
    s, e = orc.compute_range([10.0], [0.0, 1.0], 0.5)
    assert (s[0], e[0]) == (1, 1) and abs(10.0 - 1.0) > 0.5
    s, e = orc.compute_range([0.0], [5.0, 6.0], 1.0)
    assert (s[0], e[0]) == (0, 0) and abs(0.0 - 5.0) > 1.0


def test_compute_range_rejects_negative_eps(orc):
    with pytest.raises(ValueError):
        orc.compute_range([1.0], [1.0], -0.1)


def test_compute_range_vs_equation_11(orc):
    """1000 random instances with ties: the two-pointer prose reconstruction equals
    the declarative Eq. (11) on every non-empty row; an empty row is either
    naturally empty (s > e) or gets a one-element convenience range at 0 or
    Nj - 1 whose element fails the check."""
    rng = np.random.default_rng(0)
    for _ in range(1000):
        m, n = rng.integers(1, 40), rng.integers(1, 40)
        sa = np.sort(np.round(rng.uniform(0, 100, m), 0 if rng.random() < 0.3 else 3))
        sb = np.sort(np.round(rng.uniform(0, 100, n), 0 if rng.random() < 0.3 else 3))
        eps = float(rng.uniform(0, 20))
        s, e = orc.compute_range(sa, sb, eps)
        s0, e0 = orc.ranges_definition(sa, sb, eps)
        for i in range(m):
            if s0[i] <= e0[i]:
                assert (s[i], e[i]) == (s0[i], e0[i])
            else:
                # either naturally empty (s > e) or a convenience range at an end
                assert s[i] > e[i] or (s[i] == e[i] and s[i] in (0, n - 1)
                                       and abs(sa[i] - sb[s[i]]) > eps)
        # Lemma 2 (Eq. se2): monotone ranges over non-empty rows
        ne = s0 <= e0
        assert np.all(np.diff(s0[ne]) >= 0) and np.all(np.diff(e0[ne]) >= 0)


def test_lemma1_lower_bound_random(orc):
    """dist(a, b) >= |dist(p, a) - dist(p, b)| for both norms (Lemma 1)."""
    rng = np.random.default_rng(1)
    for d in (2, 64):
        A = rng.normal(size=(2000, d))
        B = rng.normal(size=(2000, d))
        P = rng.normal(size=(2000, d)) * 3
        for norm in (1, 2):
            ab = np.linalg.norm(A - B, ord=norm, axis=1)
            pa = np.array([orc.pivot_distances(A[i:i + 1], P[i], norm)[0] for i in range(0, 2000, 50)])
            pb = np.array([orc.pivot_distances(B[i:i + 1], P[i], norm)[0] for i in range(0, 2000, 50)])
            assert np.all(ab[::50] >= np.abs(pa - pb) - 1e-12 * (1 + np.abs(pa) + np.abs(pb)))


def test_pivot_distance_closed_forms(orc):
    eye = np.eye(5)
    assert np.allclose(orc.pivot_distances(eye, np.zeros(5), 2), 1.0)
    assert np.allclose(orc.pivot_distances(eye, np.zeros(5), 1), 1.0)
    assert np.allclose(orc.pivot_distances(eye, np.ones(5), 1), 4.0)
    assert np.allclose(orc.pivot_distances(eye, np.ones(5), 2), 2.0)
    assert orc.pivot_distances(np.zeros((0, 5)), np.zeros(5), 2).shape == (0,)


def test_sort_side_contract(orc):
    perm, srt = orc.sort_side([3.0, 1.0, 2.0])
    assert perm.tolist() == [1, 2, 0] and srt.tolist() == [1.0, 2.0, 3.0]
    perm, _ = orc.sort_side([1.0, 1.0, 1.0])
    assert perm.tolist() == [0, 1, 2]


def test_grouping_paper_example(orc, golden):
    for ex in golden["grouping"]:
        got = orc.group_candidates(np.array(ex["s"]), np.array(ex["e"]), ex["max_group_size"])
        assert [list(g) for g in got] == ex["groups"], ex["cite"]


def test_filtered_join_equals_brute_force(orc):
    """Fig. algo1 end to end in plain numpy: per relation, pivot distances, sort,
    compute_range, verify only [s_i, e_i] -- returns exactly the brute-force set
    (Lemma 1 + 2 make the filter lossless)."""
    E, Rel = generate(300, 4, 12, seed=21)
    for norm in (1, 2):
        eps = 1.3 if norm == 2 else 3.0
        truth = {(int(a), int(b), int(c)) for a, b, c in
                 zip(*[orc.join(E, Rel, norm, eps)[f] for f in ("h", "r", "t")])}
        got = set()
        p = np.zeros(E.shape[1])
        B = E.astype(np.float64)
        pb, sbv = orc.sort_side(orc.pivot_distances(B, p, norm))
        for r in range(Rel.shape[0]):
            A = orc.connector1(E, Rel[r])
            pa, sav = orc.sort_side(orc.pivot_distances(A, p, norm))
            s, e = orc.compute_range(sav, sbv, eps)
            for i in range(len(pa)):
                for j in range(s[i], e[i] + 1):
                    h, t = int(pa[i]), int(pb[j])
                    if orc.dist3(E[h], Rel[r], E[t], norm) <= eps:
                        got.add((h, r, t))
        assert got == truth
