"""GPU Structured Embedding join (kgc_join_se, PAPER.md:193 SE)
against the oracle's FP64 brute force (oracle.se_join) on the same seeded inputs,
through the C ABI."""
import numpy as np
import pytest

from oracle import oracle as orc
from synth import generate_se

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2307_12059_b200 import _build
    _build.build()


def _se_theta(E, Wl, Wr, hit):
    A, B = orc.se_connectors(E, Wl, Wr)
    D = np.sort(np.abs(A[0][:64, None, :] - B[0][None, :, :]).sum(axis=2).ravel())
    k = max(1, int(hit * D.size))
    return float(np.float32(0.5 * (D[k] + D[k + 1])))


def _gpu_se(E, Wl, Wr, eps, device=True, **opts):
    import torch

    from paper_2307_12059_b200 import kgc
    with kgc.Join(**opts) as j:
        if device:
            args = [torch.from_numpy(np.ascontiguousarray(x)).cuda() for x in (E, Wl, Wr)]
        else:
            args = [np.ascontiguousarray(x) for x in (E, Wl, Wr)]
        j.run_se(*args, eps)
        return j.results(), j.stats()


def _check(E, Wl, Wr, eps, res, band=1e-4, dist_rel=1e-5):
    loose = orc.se_join(E, Wl, Wr, eps * (1 + band))
    key = lambda a: set(zip(a["h"].tolist(), a["r"].tolist(), a["t"].tolist()))  # noqa: E731
    g, lo = key(res), key(loose)
    assert len(g) == res.size                      # no duplicates
    assert g <= lo                                 # nothing beyond the band
    tight = {k for k, d in zip(zip(loose["h"].tolist(), loose["r"].tolist(), loose["t"].tolist()), loose["dist"])
             if d < eps * (1 - band)}
    assert tight <= g                              # nothing missed
    ref = {k: d for k, d in zip(zip(loose["h"].tolist(), loose["r"].tolist(), loose["t"].tolist()), loose["dist"])}
    for (h, r, t), d in zip(zip(res["h"].tolist(), res["r"].tolist(), res["t"].tolist()), res["dist"]):
        assert abs(float(d) - ref[(h, r, t)]) <= dist_rel * max(ref[(h, r, t)], eps)
    return len(tight)


@pytest.mark.parametrize("N,R,d", [(300, 3, 16), (257, 2, 50), (129, 4, 100), (70, 2, 300)])
@pytest.mark.parametrize("dist", ["cluster", "uniform"])
def test_se_vs_oracle(N, R, d, dist):
    E, Wl, Wr = generate_se(N, R, d, seed=N + d, dist=dist)
    eps = _se_theta(E, Wl, Wr, 0.01)
    res, st = _gpu_se(E, Wl, Wr, eps)
    assert _check(E, Wl, Wr, eps, res) > 0
    assert st["results"] == res.size and st["R"] == R


@pytest.mark.parametrize("pivots", [1, 8])
def test_se_pivots_and_host_inputs(pivots):
    E, Wl, Wr = generate_se(600, 3, 32, seed=9)
    eps = _se_theta(E, Wl, Wr, 0.005)
    a, _ = _gpu_se(E, Wl, Wr, eps, pivots=pivots)
    b, _ = _gpu_se(E, Wl, Wr, eps, device=False, pivots=pivots)
    _check(E, Wl, Wr, eps, a)
    assert set(zip(a["h"].tolist(), a["r"].tolist(), a["t"].tolist())) == \
        set(zip(b["h"].tolist(), b["r"].tolist(), b["t"].tolist()))


def test_se_planted_and_errors():
    from paper_2307_12059_b200 import kgc
    E = np.array([[0.5, 1.0], [1.0, 2.0], [3.0, -1.0]], np.float32)
    Wl = np.array([2 * np.eye(2)], np.float32)
    Wr = np.array([np.eye(2)], np.float32)
    res, _ = _gpu_se(E, Wl, Wr, 0.0)
    assert {(int(h), int(t)) for h, t in zip(res["h"], res["t"])} == {(0, 1)} and res["dist"][0] == 0
    with kgc.Join() as j:
        with pytest.raises(kgc.KgcError):
            kgc.kgc_join_se(j.ctx, E, Wl, Wr, 3, 1, 2, -1.0)
        E2 = E.copy()
        E2[0, 0] = np.nan
        with pytest.raises(kgc.KgcError):
            kgc.kgc_join_se(j.ctx, E2, Wl, Wr, 3, 1, 2, 0.5)
