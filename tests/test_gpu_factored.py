"""GPU parity of the relation-factored L2 engine (l2_engine 5):
D^2(h, r, t) = ||h + r||^2 + ||t||^2 - 2 h.t - 2 r.t (TransE), so one tensor-core
tile of G = H T^T serves every relation; the epilogue adds r.t and tests against
(||h + r||^2 - theta^2) / 2 with a rigorous band, and the FP64 re-check decides."""
import numpy as np
import pytest

from synth import generate, generate_config, sample_rows
from tests.gpu_util import check_parity, gpu_join, keyset, theta_for

pytestmark = pytest.mark.gpu

FACT = dict(l2_engine=5)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2307_12059_b200 import _build
    _build.build()


@pytest.mark.parametrize("dist", ["cluster", "uniform"])
def test_factored_c1_full(dist):
    E, Rel = generate(1000, 10, 50, seed=1, dist=dist)
    eps = theta_for(E, Rel, 2, 1e-3)
    res, st = gpu_join(E, Rel, 2, eps, **FACT)
    assert st["engine"] == 7
    assert st["tile_pairs_total"] == 8 * 4  # relation-independent tiles: ceil(1000/128) x ceil(1000/256)
    rep = check_parity(E, Rel, 2, eps, res)
    assert rep["tight"] > 1000


@pytest.mark.parametrize("N,R,d", [(1, 1, 1), (7, 3, 5), (129, 2, 9), (257, 3, 33), (300, 5, 100), (1000, 4, 200),
                                   (513, 2, 256), (700, 3, 50), (2049, 7, 104)])
@pytest.mark.parametrize("dist", ["cluster", "uniform"])
def test_factored_ragged(N, R, d, dist):
    E, Rel = generate(N, R, d, seed=7 * N + d, dist=dist)
    eps = theta_for(E, Rel, 2, 0.01 if N > 10 else 0.3)
    res, st = gpu_join(E, Rel, 2, eps, **FACT)
    assert st["engine"] == 7
    check_parity(E, Rel, 2, eps, res)


def test_factored_equals_pruned_tiles():
    E, Rel = generate(6000, 9, 64, seed=71, dist="uniform")
    eps = theta_for(E, Rel, 2, 1e-3)
    a, _ = gpu_join(E, Rel, 2, eps, l2_engine=1)
    b, sb = gpu_join(E, Rel, 2, eps, **FACT)
    assert sb["engine"] == 7 and keyset(a) == keyset(b)


@pytest.mark.parametrize("world", [2, 3])
def test_factored_sharding_invariance(world):
    E, Rel = generate(3000, 6, 48, seed=72, dist="uniform")
    eps = theta_for(E, Rel, 2, 1e-3)
    full, _ = gpu_join(E, Rel, 2, eps, **FACT)
    parts = [gpu_join(E, Rel, 2, eps, rank=r, world=world, **FACT)[0] for r in range(world)]
    sets = [keyset(p) for p in parts]
    assert sum(len(s) for s in sets) == len(set().union(*sets))
    assert set().union(*sets) == keyset(full)


def test_factored_host_inputs_capacity_and_errors():
    from paper_2307_12059_b200 import kgc
    E, Rel = generate(2000, 4, 40, seed=73)
    eps = theta_for(E, Rel, 2, 3e-3)
    a, sa = gpu_join(E, Rel, 2, eps, device_inputs=False, result_capacity=16, **FACT)
    assert sa["reruns"] >= 1
    check_parity(E, Rel, 2, eps, a)
    bad = E.copy()
    bad[5, 3] = np.nan
    with kgc.Join(**FACT) as j:
        with pytest.raises(kgc.KgcError):
            j.run(bad, Rel, 2, eps)


@pytest.mark.parametrize("cfg,hit,S", [("c2", 1e-4, 600), ("c3", 1e-5, 400)])
def test_factored_full_size_sampled(cfg, hit, S):
    E, Rel = generate_config(cfg)
    N, R = E.shape[0], Rel.shape[0]
    rows = sample_rows(N, R, S, seed=11)
    eps = theta_for(E, Rel, 2, hit, rows=rows)
    res, st = gpu_join(E, Rel, 2, eps, **FACT)
    assert st["engine"] == 7
    rep = check_parity(E, Rel, 2, eps, res, rows=rows)
    assert rep["tight"] > 0
