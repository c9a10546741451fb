"""Negative pins for oracle.compare, the checker every GPU parity test relies on
(no GPU).  The comparator implements the north_star's parity bar (BASELINE.json:
the exact set outside |dist - theta| <= 1e-4 theta, distances within 1e-5
relative; SURVEY.md §8(c) "Comparator"): tight <= gpu <= loose, no duplicates,
|d_gpu - d_orc| <= 1e-5 max(d_orc, theta).  Each test injects one plausible GPU
mistake into an otherwise exact copy of the oracle's own answer and checks that
compare() flags it -- and that the don't-care band really is don't-care.
"""
import numpy as np
import pytest

from synth import generate

EPS_BAND = 1e-4


@pytest.fixture(scope="module")
def case(orc):
    E, Rel = generate(300, 4, 16, seed=11)
    rows = np.arange(300 * 4)
    eps, _ = orc.calibrate_theta(E, Rel, 2, 5e-3, rows)
    loose = orc.join(E, Rel, 2, eps * (1 + EPS_BAND))
    tight = loose[loose["dist"] < eps * (1 - EPS_BAND)]
    assert tight.size > 100
    return eps, loose, tight


def _ok(orc, gpu, loose, eps):
    return orc.compare(gpu, loose, eps, band_rel=EPS_BAND, dist_rel=1e-5)


def test_exact_copy_passes(orc, case):
    eps, loose, tight = case
    rep = _ok(orc, tight.copy(), loose, eps)
    assert rep["ok"] and rep["missing"] == rep["extra"] == rep["duplicates"] == 0


def test_band_members_are_dont_care(orc, case):
    """Records with theta(1 - 1e-4) <= dist <= theta(1 + 1e-4) may be present or absent."""
    eps, loose, tight = case
    assert _ok(orc, loose.copy(), loose, eps)["ok"]      # all band members reported
    assert _ok(orc, tight.copy(), loose, eps)["ok"]      # none reported


def test_dropped_record_fails(orc, case):
    eps, loose, tight = case
    g = np.delete(tight.copy(), tight.size // 2)
    rep = _ok(orc, g, loose, eps)
    assert not rep["ok"] and rep["missing"] == 1


def test_duplicated_record_fails(orc, case):
    eps, loose, tight = case
    g = np.concatenate([tight, tight[:1]])
    rep = _ok(orc, g, loose, eps)
    assert not rep["ok"] and rep["duplicates"] == 1


@pytest.mark.parametrize("field", ["h", "r", "t"])
def test_wrong_index_fails(orc, case, field):
    """A transposed or off-by-one index turns a true record into a false one (extra) and
    loses the true one (missing)."""
    eps, loose, tight = case
    g = tight.copy()
    i = g.size // 3
    n = 300 if field in ("h", "t") else 4
    g[field][i] = (g[field][i] + 1) % n
    rep = _ok(orc, g, loose, eps)
    assert not rep["ok"]
    assert rep["missing"] >= 1 or rep["duplicates"] >= 1


def test_record_outside_loose_fails(orc, case):
    eps, loose, tight = case
    far = orc.join(*generate(300, 4, 16, seed=11), 2, eps * 1.5)
    extra = far[far["dist"] > eps * (1 + 2 * EPS_BAND)][:1]
    assert extra.size == 1
    rep = _ok(orc, np.concatenate([tight, extra]), loose, eps)
    assert not rep["ok"] and rep["extra"] == 1


@pytest.mark.parametrize("rel", [1.5e-5, 1e-4, 1e-2])
def test_distance_perturbation_fails(orc, case, rel):
    """A reported distance off by more than 1e-5 relative (of max(d, theta)) is flagged."""
    eps, loose, tight = case
    g = tight.copy()
    i = int(np.argmax(g["dist"]))
    g["dist"][i] = np.float32(g["dist"][i] + rel * max(float(g["dist"][i]), eps))
    rep = _ok(orc, g, loose, eps)
    assert not rep["ok"] and rep["max_dist_rel_err"] > 1e-5


def test_distance_within_tolerance_passes(orc, case):
    eps, loose, tight = case
    g = tight.copy()
    g["dist"] = (g["dist"].astype(np.float64) * (1 + 5e-6)).astype(np.float32)
    assert _ok(orc, g, loose, eps)["ok"]
