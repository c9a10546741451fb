"""GPU parity of the gathered-tail SIMT engine (engine 5, l1_engine 3): inside
every surviving tile pair only the tails whose own K pivot keys pass Lemma 1's
L_inf test against the query tile's key box are computed (pivots.cu,
tiles_simt.cu).  Lemma 1 makes the dropped tails provably
farther than theta from every query of the tile, so the set must not change."""
import numpy as np
import pytest

from synth import generate, generate_config, sample_rows
from tests.gpu_util import check_parity, gpu_join, keyset, theta_for

pytestmark = pytest.mark.gpu

L1_GATHER = dict(pivots=8, l1_engine=3)
L1_TILES = dict(pivots=8, l1_engine=2)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2307_12059_b200 import _build
    _build.build()


@pytest.mark.parametrize("norm", [1, 2])
@pytest.mark.parametrize("K", [2, 8])
def test_gather_c1_full(norm, K):
    E, Rel = generate_config("c1")
    eps = theta_for(E, Rel, norm, 1e-3)
    opts = dict(pivots=K, l1_engine=3, l2_engine=2)
    res, st = gpu_join(E, Rel, norm, eps, **opts)
    assert st["engine"] == 5 and st["pivots_used"] == K
    rep = check_parity(E, Rel, norm, eps, res)
    assert rep["tight"] > 1000
    assert 0 < st["gathered_pairs"] < st["tile_pairs_surviving"] * 64 * 64


def test_gather_is_l1_default_with_pivots():
    E, Rel = generate_config("c1")
    eps = theta_for(E, Rel, 1, 1e-3)
    _, st = gpu_join(E, Rel, 1, eps, pivots=8)
    assert st["engine"] == 5
    _, st1 = gpu_join(E, Rel, 1, eps)           # one pivot: contiguous tiles
    assert st1["engine"] == 2


@pytest.mark.parametrize("N,R,d", [(1, 1, 1), (7, 3, 5), (65, 2, 8), (129, 2, 9), (300, 5, 100), (1000, 4, 200),
                                   (513, 2, 256), (700, 3, 50), (2049, 3, 33)])
@pytest.mark.parametrize("norm", [1, 2])
@pytest.mark.parametrize("dist", ["cluster", "uniform"])
def test_gather_ragged(N, R, d, norm, dist):
    E, Rel = generate(N, R, d, seed=3 * N + d, dist=dist)
    eps = theta_for(E, Rel, norm, 0.01 if N > 10 else 0.3)
    res, st = gpu_join(E, Rel, norm, eps, pivots=8, l1_engine=3, l2_engine=2)
    assert st["engine"] == (5 if st["work_items_mine"] > 0 else 2)
    check_parity(E, Rel, norm, eps, res)


@pytest.mark.parametrize("norm", [1, 2])
def test_gather_equals_contiguous_tiles(norm):
    E, Rel = generate(8000, 5, 64, seed=51)
    eps = theta_for(E, Rel, norm, 1e-3)
    a, sa = gpu_join(E, Rel, norm, eps, pivots=8, l1_engine=2, l2_engine=2)
    b, sb = gpu_join(E, Rel, norm, eps, pivots=8, l1_engine=3, l2_engine=2)
    assert sa["engine"] == 2 and sb["engine"] == 5
    assert keyset(a) == keyset(b)
    assert sa["tile_pairs_surviving"] == sb["tile_pairs_surviving"]
    assert sb["gathered_pairs"] < sb["tile_pairs_surviving"] * 64 * 64
    # same candidates up to tails dropped by the per-tail test (all provably misses)
    assert sb["candidates"] <= sa["candidates"]


def test_gather_lists_complete_and_sound():
    """Every (query tile, tail) with some query row passing the K-pivot L_inf
    test (|d(p_k,q) - d(p_k,t)| <= eps for all k) is in the query tile's
    gathered list; lists are ascending, padded with N to blocks of 64, and hold
    only tails of the query tile's surviving tiles."""
    from paper_2307_12059_b200 import kgc
    N, R, K, d = 3000, 3, 8, 32
    E, Rel = generate(N, R, d, seed=52)
    eps = theta_for(E, Rel, 1, 1e-3)
    with kgc.Join(pivots=K, l1_engine=3) as j:
        j.run(E, Rel, 1, eps)
        kt = j.inspect("tail_keys").reshape(N, K)
        kq = j.inspect("query_keys").reshape(R, N, K)
        tperm = j.inspect("tail_perm")
        qperm = j.inspect("query_perm").reshape(R, N)
        cum = j.inspect("query_cost")
        lst = j.inspect("tile_list")
        gcum = j.inspect("gather_cost")
        glist = j.inspect("gather_list")
        st = j.stats()
    assert st["engine"] == 5
    BM, BN, QT = st["query_tile_rows"], st["tail_tile_rows"], st["query_tiles"]
    skt = kt[tperm]
    nq = R * QT
    assert gcum.shape == (nq,) and len(glist) == 64 * len(lst)
    for r in range(R):
        skq = kq[r][qperm[r]]
        for qt in range(QT):
            tq = r * QT + qt
            ntl = (cum[tq + 1] if tq + 1 < nq else len(lst) + cum[0]) - cum[tq]
            g0 = 64 * (cum[tq] - cum[0])
            seg = glist[g0:g0 + 64 * gcum[tq]]
            assert gcum[tq] <= ntl
            real = seg[seg < N]
            assert len(seg) == 64 * ((len(real) + 63) // 64)      # whole blocks
            assert np.all(seg[len(real):] == N)                  # padding at the end only
            assert np.all(np.diff(real) > 0)                      # ascending, unique
            tiles = set(lst[cum[tq] - cum[0]: cum[tq] - cum[0] + ntl].tolist())
            assert set((real // BN).tolist()) <= tiles
            rows = skq[qt * BM:(qt + 1) * BM]
            ok = np.ones((rows.shape[0], N), bool)
            for k in range(K):
                ok &= np.abs(rows[:, None, k] - skt[None, :, k]) <= eps
            need = set(np.nonzero(ok.any(axis=0))[0].tolist())
            assert need <= set(real.tolist())
    assert st["gathered_pairs"] == BM * int(np.sum([np.sum(glist[64 * (cum[q] - cum[0]):][:64 * gcum[q]] < N)
                                                     for q in range(nq)]))


@pytest.mark.parametrize("world", [2, 3, 5])
def test_gather_sharding_invariance(world):
    E, Rel = generate(4000, 7, 48, seed=53)
    eps = theta_for(E, Rel, 1, 1e-3)
    full, _ = gpu_join(E, Rel, 1, eps, **L1_GATHER)
    for split in (0, 1, 2):
        parts = [gpu_join(E, Rel, 1, eps, rank=r, world=world, split=split, **L1_GATHER)[0] for r in range(world)]
        sets = [keyset(p) for p in parts]
        assert sum(len(s) for s in sets) == len(set().union(*sets))
        assert set().union(*sets) == keyset(full)


def test_gather_host_inputs_and_capacity_rerun():
    E, Rel = generate(3000, 4, 40, seed=54)
    eps = theta_for(E, Rel, 1, 3e-3)
    a, sa = gpu_join(E, Rel, 1, eps, device_inputs=False, result_capacity=16, **L1_GATHER)
    b, _ = gpu_join(E, Rel, 1, eps, **L1_GATHER)
    assert sa["reruns"] >= 1
    assert keyset(a) == keyset(b)
    check_parity(E, Rel, 1, eps, a)


@pytest.mark.parametrize("hit", [1e-5, 1e-4])
def test_gather_c2_l1_full_size_sampled(hit):
    E, Rel = generate_config("c2")
    N, R = E.shape[0], Rel.shape[0]
    rows = sample_rows(N, R, 1200, seed=9)
    eps = theta_for(E, Rel, 1, hit, rows=rows)
    res, st = gpu_join(E, Rel, 1, eps, **L1_GATHER)
    assert st["engine"] == 5
    rep = check_parity(E, Rel, 1, eps, res, rows=rows)
    assert rep["tight"] > 0


# ------------------------------------------------- tensor-core engine on gathered tail blocks (l2_engine 4)
TC_GATHER = dict(pivots=8, l2_engine=4)


@pytest.mark.parametrize("K", [2, 8])
def test_tc_gather_c1_full(K):
    E, Rel = generate_config("c1")
    eps = theta_for(E, Rel, 2, 1e-3)
    res, st = gpu_join(E, Rel, 2, eps, pivots=K, l2_engine=4)
    assert st["engine"] == 6 and st["pivots_used"] == K
    assert st["query_tile_rows"] == 128 and st["tail_tile_rows"] == 256
    rep = check_parity(E, Rel, 2, eps, res)
    assert rep["tight"] > 1000
    assert 0 < st["gathered_pairs"] <= st["tile_pairs_surviving"] * 128 * 256


@pytest.mark.parametrize("N,R,d", [(1, 1, 1), (7, 3, 5), (129, 2, 9), (257, 3, 33), (300, 5, 100), (1000, 4, 200),
                                   (513, 2, 256), (700, 3, 50), (3000, 3, 8), (2049, 2, 104)])
@pytest.mark.parametrize("dist", ["cluster", "uniform"])
def test_tc_gather_ragged(N, R, d, dist):
    E, Rel = generate(N, R, d, seed=5 * N + d, dist=dist)
    eps = theta_for(E, Rel, 2, 0.01 if N > 10 else 0.3)
    res, st = gpu_join(E, Rel, 2, eps, **TC_GATHER)
    assert st["engine"] == (6 if st["work_items_mine"] > 0 else 1)
    check_parity(E, Rel, 2, eps, res)


def test_tc_gather_equals_contiguous_tiles():
    E, Rel = generate(12000, 5, 64, seed=61)
    eps = theta_for(E, Rel, 2, 1e-3)
    a, sa = gpu_join(E, Rel, 2, eps, pivots=8, l2_engine=1)
    b, sb = gpu_join(E, Rel, 2, eps, **TC_GATHER)
    assert sa["engine"] == 1 and sb["engine"] == 6
    assert keyset(a) == keyset(b)
    assert sa["tile_pairs_surviving"] == sb["tile_pairs_surviving"]
    assert sb["gathered_pairs"] < sb["tile_pairs_surviving"] * 128 * 256
    assert sb["candidates"] <= sa["candidates"] * 1.05 + 100


def test_tc_gather_lists_complete():
    from paper_2307_12059_b200 import kgc
    N, R, K, d = 4000, 3, 8, 32
    E, Rel = generate(N, R, d, seed=62)
    eps = theta_for(E, Rel, 2, 1e-3)
    with kgc.Join(**TC_GATHER) as j:
        j.run(E, Rel, 2, eps)
        kt = j.inspect("tail_keys").reshape(N, K)
        kq = j.inspect("query_keys").reshape(R, N, K)
        tperm = j.inspect("tail_perm")
        qperm = j.inspect("query_perm").reshape(R, N)
        cum = j.inspect("query_cost")
        lst = j.inspect("tile_list")
        nb = j.inspect("gather_cost")
        glist = j.inspect("gather_list")
        st = j.stats()
    assert st["engine"] == 6
    BM, BN, QT = st["query_tile_rows"], st["tail_tile_rows"], st["query_tiles"]
    skt = kt[tperm]
    nq = R * QT
    assert len(glist) == BN * len(lst)
    total = 0
    for r in range(R):
        skq = kq[r][qperm[r]]
        for qt in range(QT):
            tq = r * QT + qt
            ntl = (cum[tq + 1] if tq + 1 < nq else len(lst) + cum[0]) - cum[tq]
            seg = glist[BN * (cum[tq] - cum[0]):][:BN * nb[tq]]
            real = seg[seg < N]
            total += len(real)
            assert len(seg) == BN * ((len(real) + BN - 1) // BN)
            assert np.all(seg[len(real):] == N) and np.all(np.diff(real) > 0)
            tiles = set(lst[cum[tq] - cum[0]: cum[tq] - cum[0] + ntl].tolist())
            assert set((real // BN).tolist()) <= tiles
            rows = skq[qt * BM:(qt + 1) * BM]
            ok = np.ones((rows.shape[0], N), bool)
            for k in range(K):
                ok &= np.abs(rows[:, None, k] - skt[None, :, k]) <= eps
            assert set(np.nonzero(ok.any(axis=0))[0].tolist()) <= set(real.tolist())
    assert st["gathered_pairs"] == BM * total


@pytest.mark.parametrize("world", [2, 3])
def test_tc_gather_sharding_invariance(world):
    E, Rel = generate(5000, 7, 48, seed=63)
    eps = theta_for(E, Rel, 2, 1e-3)
    full, _ = gpu_join(E, Rel, 2, eps, **TC_GATHER)
    for split in (0, 1, 2):
        parts = [gpu_join(E, Rel, 2, eps, rank=r, world=world, split=split, **TC_GATHER)[0] for r in range(world)]
        sets = [keyset(p) for p in parts]
        assert sum(len(s) for s in sets) == len(set().union(*sets))
        assert set().union(*sets) == keyset(full)


@pytest.mark.parametrize("cfg,hit,S", [("c2", 1e-4, 1200), ("c3", 1e-5, 800), ("c3", 1e-3, 400)])
def test_tc_gather_full_size_sampled(cfg, hit, S):
    E, Rel = generate_config(cfg)
    N, R = E.shape[0], Rel.shape[0]
    rows = sample_rows(N, R, S, seed=10)
    eps = theta_for(E, Rel, 2, hit, rows=rows)
    res, st = gpu_join(E, Rel, 2, eps, **TC_GATHER)
    assert st["engine"] == 6
    rep = check_parity(E, Rel, 2, eps, res, rows=rows)
    assert rep["tight"] > 0


# ------------------------------------------------- CTA-pair tensor-core engine on gathered blocks (l2_engine 6)
TC2_GATHER = dict(pivots=8, l2_engine=6)


@pytest.mark.parametrize("K", [2, 8])
def test_tc2_gather_c1_full(K):
    E, Rel = generate_config("c1")
    eps = theta_for(E, Rel, 2, 1e-3)
    res, st = gpu_join(E, Rel, 2, eps, pivots=K, l2_engine=6)
    assert st["engine"] == 8 and st["pivots_used"] == K
    assert st["query_tile_rows"] == 256 and st["tail_tile_rows"] == 256
    rep = check_parity(E, Rel, 2, eps, res)
    assert rep["tight"] > 1000
    assert 0 < st["gathered_pairs"] <= st["tile_pairs_surviving"] * 256 * 256


def test_tc2_gather_one_pivot_is_contiguous_pair_engine():
    E, Rel = generate_config("c1")
    eps = theta_for(E, Rel, 2, 1e-3)
    res, st = gpu_join(E, Rel, 2, eps, pivots=1, l2_engine=6)
    assert st["engine"] == 4
    check_parity(E, Rel, 2, eps, res)


@pytest.mark.parametrize("N,R,d", [(1, 1, 1), (7, 3, 5), (129, 2, 9), (257, 3, 33), (300, 5, 100), (1000, 4, 200),
                                   (513, 2, 256), (700, 3, 50), (3000, 3, 8), (2049, 2, 104), (5000, 2, 36)])
@pytest.mark.parametrize("dist", ["cluster", "uniform"])
def test_tc2_gather_ragged(N, R, d, dist):
    E, Rel = generate(N, R, d, seed=7 * N + d, dist=dist)
    eps = theta_for(E, Rel, 2, 0.01 if N > 10 else 0.3)
    res, st = gpu_join(E, Rel, 2, eps, **TC2_GATHER)
    assert st["engine"] in (8, 4)
    check_parity(E, Rel, 2, eps, res)


def test_tc2_gather_equals_contiguous_pair_tiles():
    E, Rel = generate(12000, 5, 64, seed=61)
    eps = theta_for(E, Rel, 2, 1e-3)
    a, sa = gpu_join(E, Rel, 2, eps, pivots=8, l2_engine=3)
    b, sb = gpu_join(E, Rel, 2, eps, **TC2_GATHER)
    assert sa["engine"] == 4 and sb["engine"] == 8
    assert keyset(a) == keyset(b)
    assert sa["tail_tile_rows"] == 128 and sb["tail_tile_rows"] == 256  # contiguous pair tiles are 128 tails
    assert sb["gathered_pairs"] < sb["tile_pairs_surviving"] * 256 * 256


@pytest.mark.parametrize("world", [2, 3])
def test_tc2_gather_sharding_invariance(world):
    E, Rel = generate(5000, 7, 48, seed=64)
    eps = theta_for(E, Rel, 2, 1e-3)
    full, _ = gpu_join(E, Rel, 2, eps, **TC2_GATHER)
    for split in (0, 1, 2):
        parts = [gpu_join(E, Rel, 2, eps, rank=r, world=world, split=split, **TC2_GATHER)[0] for r in range(world)]
        sets = [keyset(p) for p in parts]
        assert sum(len(s) for s in sets) == len(set().union(*sets))
        assert set().union(*sets) == keyset(full)


def test_tc2_gather_host_inputs_and_capacity_rerun():
    E, Rel = generate(6000, 4, 40, seed=65)
    eps = theta_for(E, Rel, 2, 2e-3)
    a, sa = gpu_join(E, Rel, 2, eps, device_inputs=False, result_capacity=16, **TC2_GATHER)
    assert sa["reruns"] >= 1 and sa["engine"] == 8
    check_parity(E, Rel, 2, eps, a)


@pytest.mark.parametrize("cfg,hit,S", [("c2", 1e-4, 1200), ("c3", 1e-5, 800), ("c4", 1e-5, 300), ("c3", 1e-3, 300)])
def test_tc2_gather_full_size_sampled(cfg, hit, S):
    E, Rel = generate_config(cfg)
    N, R = E.shape[0], Rel.shape[0]
    rows = sample_rows(N, R, S, seed=11)
    eps = theta_for(E, Rel, 2, hit, rows=rows)
    res, st = gpu_join(E, Rel, 2, eps, **TC2_GATHER)
    assert st["engine"] == 8
    rep = check_parity(E, Rel, 2, eps, res, rows=rows)
    assert rep["tight"] > 0


@pytest.mark.parametrize("offset", [0.0, 1000.0])
@pytest.mark.parametrize("K", [3, 8, 16, 32, 64, 128])
def test_l2_factorised_keys_accuracy(offset, K):
    """L2 K-pivot keys come from the FP64 factorisation ||h + r - p||^2 = ||h - p||^2 +
    2 h.r - 2 r.p + ||r||^2 (pivots.cu, mp_qkeys_fact_kernel): each key is within 2^-21
    relative (fl32 rounding of D^2 and the hardware sqrt approximation) + delta_r = sqrt((d + 8) 2^-53)(max||h|| + ||r|| + max||p||) of the exact
    distance from the EXACT h + r (pivot_distances in FP64 on h + r formed in FP64), and the
    tail keys within 2^-21 relative of d(p_k, t); the tile test's margin is (d + 8) 2^-23 >= 9 2^-23.  The offset case (||h|| ~ 1000 sqrt(d))
    exercises the cancellation the delta term bounds."""
    from oracle import oracle as orc
    from paper_2307_12059_b200 import kgc
    N, R, d = 1500, 5, 48
    E, Rel = generate(N, R, d, seed=77 + K)
    E = (E.astype(np.float64) + offset).astype(np.float32)
    eps = theta_for(E, Rel, 2, 1e-3)
    with kgc.Join(pivots=K, l2_engine=1) as j:
        j.run(E, Rel, 2, eps)
        P = j.inspect("pivots").reshape(K, d)
        kt = j.inspect("tail_keys").reshape(N, K)
        kq = j.inspect("query_keys").reshape(R, N, K)
        assert j.stats()["pivots_used"] == K
    E64, R64 = E.astype(np.float64), Rel.astype(np.float64)
    hmax = np.sqrt((E64 ** 2).sum(1)).max()
    pmax = np.sqrt((P.astype(np.float64) ** 2).sum(1)).max()
    # tail keys from the GEMM-form entity terms: within 2^-21 relative + delta_t (pivots.cu)
    delta_t = np.sqrt((d + 4) * 2.0 ** -53) * (hmax + pmax)
    for k in range(K):
        exact_t = orc.pivot_distances(E64, P[k], 2)
        assert np.all(np.abs(kt[:, k] - exact_t) <= 2 ** -21 * exact_t + delta_t)
        for r in range(R):
            exact_q = orc.pivot_distances(E64 + R64[r][None, :], P[k], 2)
            delta = np.sqrt((d + 8) * 2.0 ** -53) * (hmax + np.linalg.norm(R64[r]) + pmax)
            err = np.abs(kq[r, :, k].astype(np.float64) - exact_q)
            assert np.all(err <= 2 ** -21 * exact_q + delta), (k, r, err.max(), delta)
    # and the join over these keys is exact
    res, st = gpu_join(E, Rel, 2, eps, pivots=K, l2_engine=1)
    check_parity(E, Rel, 2, eps, res)


@pytest.mark.parametrize("K", [12, 16, 24, 32, 48, 64, 96, 128])
@pytest.mark.parametrize("norm,opts", [(2, dict(l2_engine=1)), (2, dict(l2_engine=3)), (2, dict(l2_engine=4)),
                                       (1, dict(l1_engine=3)), (1, dict(l1_engine=2))])
def test_many_pivots_c1_full(K, norm, opts):
    if norm == 1 and K > 32:
        pytest.skip("the L1 keys support at most 32 pivots (test_pivot_count_validation)")
    """Up to 32 pivots (the tile test over all K, the per-tail test of the gathered engines over
    the first 8): the result set is the oracle's, and more pivots never keep more tile pairs."""
    E, Rel = generate_config("c1")
    eps = theta_for(E, Rel, norm, 1e-3)
    res, st = gpu_join(E, Rel, norm, eps, pivots=K, **opts)
    assert st["pivots_used"] == K
    check_parity(E, Rel, norm, eps, res)
    _, st8 = gpu_join(E, Rel, norm, eps, pivots=8, **opts)
    assert st["tile_pairs_surviving"] <= st8["tile_pairs_surviving"]


@pytest.mark.parametrize("K", [16, 32, 64, 128])
@pytest.mark.parametrize("N,R,d", [(65, 2, 8), (700, 3, 50), (2049, 3, 33), (513, 2, 256)])
def test_many_pivots_ragged(K, N, R, d):
    E, Rel = generate(N, R, d, seed=5 * N + d + K)
    for norm in ((1, 2) if K <= 32 else (2,)):
        eps = theta_for(E, Rel, norm, 0.01)
        res, st = gpu_join(E, Rel, norm, eps, pivots=K)
        check_parity(E, Rel, norm, eps, res)


def test_pivot_count_validation():
    from paper_2307_12059_b200 import kgc
    for bad in (9, 10, 17, 33, 65, 100, 129):
        with pytest.raises(Exception):
            with kgc.Join(pivots=bad) as j:
                pass
    E, Rel = generate(300, 2, 16, seed=9)
    with kgc.Join(pivots=64) as j:      # 64 pivots: L2 only
        with pytest.raises(Exception):
            j.run(E, Rel, 1, 1.0)
