"""GPU top-k (kgc_topk; PAPER.md:128's minimum-distance
statistic) against the oracle's brute force (oracle.topk) on the same seeded
inputs, through the C ABI."""
import numpy as np
import pytest

from oracle import oracle as orc
from synth import generate, generate_config, sample_rows

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2307_12059_b200 import _build
    _build.build()


def _topk(E, Rel, norm, k, exclude_self=False, device=True, **opts):
    import torch

    from paper_2307_12059_b200 import kgc
    with kgc.Join(**opts) as j:
        if device:
            Et, Rt = torch.from_numpy(E).cuda(), torch.from_numpy(Rel).cuda()
            return j.topk(Et, Rt, norm, k, exclude_self)
        return j.topk(E, Rel, norm, k, exclude_self)


def _check(got, ref, band=1e-4, dist_rel=1e-5):
    """Same length; distances within dist_rel; the sets agree outside the band around the
    k-th distance (ties near it may be ordered differently)."""
    assert got.size == ref.size
    if ref.size == 0:
        return
    dk = float(ref["dist"][-1])
    np.testing.assert_allclose(np.sort(got["dist"]).astype(np.float64), ref["dist"],
                               rtol=dist_rel, atol=dist_rel * max(dk, 1e-30))
    assert np.all(np.diff(got["dist"]) >= 0)
    g = set(zip(got["h"].tolist(), got["r"].tolist(), got["t"].tolist()))
    must = {(int(a), int(b), int(c)) for a, b, c, d in zip(ref["h"], ref["r"], ref["t"], ref["dist"])
            if d < dk * (1 - band)}
    assert must <= g
    assert len(g) == got.size  # no duplicates


@pytest.mark.parametrize("norm", [1, 2])
@pytest.mark.parametrize("exclude_self", [False, True])
@pytest.mark.parametrize("k", [1, 17, 1000])
def test_topk_small_vs_oracle(norm, exclude_self, k):
    E, Rel = generate(300, 5, 16, seed=31 + norm, dist="cluster")
    ref = orc.topk(E, Rel, norm, k, exclude_self=exclude_self)
    got = _topk(E, Rel, norm, k, exclude_self)
    _check(got, ref)


def test_topk_c1_both_engines_and_host_inputs():
    E, Rel = generate_config("c1")
    ref = orc.topk(E, Rel, 2, 50)
    for opts in (dict(l2_engine=1), dict(l2_engine=2), dict(l2_engine=3)):
        _check(_topk(E, Rel, 2, 50, **opts), ref)
    _check(_topk(E, Rel, 2, 50, device=False), ref)


def test_topk_planted_translation():
    E = np.array([[0, 0], [1, 1], [3, 0], [0.5, 2]], np.float32)
    Rel = np.array([[0, 0], [2, -1]], np.float32)      # E[1] + Rel[1] == E[2] exactly
    got = _topk(E, Rel, 2, 1, exclude_self=True)
    assert (int(got["h"][0]), int(got["r"][0]), int(got["t"][0])) == (1, 1, 2) and got["dist"][0] == 0
    got = _topk(E, Rel, 2, 5)
    assert np.all(got["dist"] == 0)


def test_topk_more_than_available():
    E, Rel = generate(5, 2, 3, seed=3)
    got = _topk(E, Rel, 1, 1000)
    assert got.size == 5 * 5 * 2
    _check(got, orc.topk(E, Rel, 1, 1000))
    got = _topk(E, Rel, 1, 1000, exclude_self=True)
    assert got.size == 5 * 4 * 2


def test_topk_errors():
    from paper_2307_12059_b200 import kgc
    E, Rel = generate(50, 2, 4, seed=1)
    with pytest.raises(kgc.KgcError):
        _topk(E, Rel, 3, 5)
    with kgc.Join(world=2, rank=0) as j:
        with pytest.raises(kgc.KgcError):
            j.topk(E, Rel, 2, 5)
    assert _topk(E, Rel, 2, 0).size == 0


@pytest.mark.parametrize("cfg,norm", [("c2", 2), ("c2", 1)])
def test_topk_full_size_sampled(cfg, norm):
    """c2-sized: every returned distance matches the oracle's for that triplet, and no
    sampled (h, r) row has a triplet closer than the k-th distance that is missing."""
    E, Rel = generate_config(cfg)
    N, R = E.shape[0], Rel.shape[0]
    k = 200
    got = _topk(E, Rel, norm, k, exclude_self=True)
    assert got.size == k
    rows = got["h"].astype(np.int64) * R + got["r"]
    D = orc.dist_rows(E, Rel, norm, rows=rows)
    d_orc = D[np.arange(k), got["t"]]
    np.testing.assert_allclose(got["dist"], d_orc, rtol=1e-5)
    dk = float(got["dist"][-1])
    srows = sample_rows(N, R, 600, seed=3)
    Ds = orc.dist_rows(E, Rel, norm, rows=srows)
    g = set(zip(got["h"].tolist(), got["r"].tolist(), got["t"].tolist()))
    for i, row in enumerate(srows):
        h, r = divmod(int(row), R)
        for t in np.nonzero(Ds[i] < dk * (1 - 1e-4))[0]:
            if t != h:
                assert (h, r, int(t)) in g
