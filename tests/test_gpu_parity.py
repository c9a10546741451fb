"""GPU parity: the CUDA path (through the C ABI) against the oracle, element by
element on the same seeded inputs (BASELINE.json north_star: exact set outside
|dist - theta| <= 1e-4 theta, distances within 1e-5 relative)."""
import numpy as np
import pytest

from oracle import oracle as orc
from synth import generate, generate_config, sample_rows
from tests.gpu_util import check_parity, gpu_join, keyset, theta_for

pytestmark = pytest.mark.gpu

ENGINES = {"tc": dict(l2_engine=1), "simt": dict(l2_engine=2), "tc2": dict(l2_engine=3)}


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2307_12059_b200 import _build
    _build.build()


# ------------------------------------------------------------ C1, full oracle
@pytest.mark.parametrize("engine", ["tc", "simt", "tc2"])
def test_c1_l2_full(engine):
    E, Rel = generate_config("c1")
    eps = theta_for(E, Rel, 2, 1e-3)
    res, st = gpu_join(E, Rel, 2, eps, **ENGINES[engine])
    rep = check_parity(E, Rel, 2, eps, res)
    assert rep["tight"] > 1000
    assert st["results"] == res.size
    assert st["triplets"] == 1000 * 1000 * 10


def test_c1_l1_full():
    E, Rel = generate_config("c1")
    eps = theta_for(E, Rel, 1, 1e-3)
    res, _ = gpu_join(E, Rel, 1, eps)
    rep = check_parity(E, Rel, 1, eps, res)
    assert rep["tight"] > 1000


# ------------------------------------------------- ragged shapes, both norms
SHAPES = [(1, 1, 1), (7, 3, 5), (129, 2, 9), (257, 3, 33), (300, 5, 100), (1000, 4, 200), (513, 2, 256),
          (600, 2, 300), (700, 3, 50)]


@pytest.mark.parametrize("N,R,d", SHAPES)
@pytest.mark.parametrize("norm", [1, 2])
@pytest.mark.parametrize("dist", ["cluster", "uniform"])
def test_ragged_shapes(N, R, d, norm, dist):
    E, Rel = generate(N, R, d, seed=N + R + d, dist=dist)
    eps = theta_for(E, Rel, norm, 0.01 if N > 10 else 0.3)
    engines = ["tc", "simt", "tc2"] if norm == 2 and d <= 256 else ["simt"]
    for eng in engines:
        res, _ = gpu_join(E, Rel, norm, eps, **ENGINES[eng])
        check_parity(E, Rel, norm, eps, res)


# ------------------------------------------------- invariances / controls
@pytest.mark.parametrize("norm", [1, 2])
def test_prune_off_gives_identical_set(norm):
    E, Rel = generate(2000, 6, 64, seed=31)
    eps = theta_for(E, Rel, norm, 1e-3)
    a, sa = gpu_join(E, Rel, norm, eps)
    b, sb = gpu_join(E, Rel, norm, eps, prune=0)
    assert keyset(a) == keyset(b)
    assert sb["tile_pairs_surviving"] == sb["tile_pairs_total"]
    assert sa["tile_pairs_surviving"] < sa["tile_pairs_total"]


@pytest.mark.parametrize("norm", [1, 2])
def test_pivot_invariance(norm):
    """Lemma 1 holds for any pivot, so the result set is pivot-invariant (reading R7)."""
    E, Rel = generate(1500, 5, 40, seed=32)
    eps = theta_for(E, Rel, norm, 1e-3)
    a, _ = gpu_join(E, Rel, norm, eps, pivot=0)
    b, _ = gpu_join(E, Rel, norm, eps, pivot=1)
    assert keyset(a) == keyset(b)
    check_parity(E, Rel, norm, eps, b)


@pytest.mark.parametrize("world,split", [(2, 0), (3, 0), (5, 0), (8, 0), (2, 1), (3, 1), (5, 1), (2, 2), (3, 2), (8, 2),
                                         (2, 3), (5, 3), (8, 3)])
def test_sharding_invariance(world, split):
    """Union of the shards of `world` contexts == the 1-context set, shards disjoint
    (split 0: rank-local preprocessing of a query-tile range; 1: global cost split; 2: cyclic)."""
    E, Rel = generate(3000, 7, 48, seed=33)
    eps = theta_for(E, Rel, 2, 1e-3)
    full, _ = gpu_join(E, Rel, 2, eps)
    parts = [gpu_join(E, Rel, 2, eps, rank=r, world=world, split=split)[0] for r in range(world)]
    sets = [keyset(p) for p in parts]
    assert sum(len(s) for s in sets) == len(set().union(*sets))
    assert set().union(*sets) == keyset(full)


@pytest.mark.parametrize("norm", [1, 2])
def test_rank_local_split_host_inputs(norm):
    """Rank-local shards with HOST inputs (the Rel sub-range is copied) == full set."""
    E, Rel = generate(1500, 9, 24, seed=46)
    eps = theta_for(E, Rel, norm, 1e-3)
    full, _ = gpu_join(E, Rel, norm, eps)
    parts = [gpu_join(E, Rel, norm, eps, device_inputs=False, rank=r, world=4)[0] for r in range(4)]
    sets = [keyset(p) for p in parts]
    assert sum(len(s) for s in sets) == len(set().union(*sets)) == len(keyset(full))
    assert set().union(*sets) == keyset(full)


def test_host_and_device_inputs_agree():
    E, Rel = generate(1200, 4, 32, seed=34)
    eps = theta_for(E, Rel, 2, 1e-3)
    a, sa = gpu_join(E, Rel, 2, eps, device_inputs=True)
    b, sb = gpu_join(E, Rel, 2, eps, device_inputs=False)
    assert keyset(a) == keyset(b)
    assert sa["h2d_bytes"] == 0 and sb["h2d_bytes"] == E.nbytes + Rel.nbytes


def test_results_into_device_buffer():
    import torch

    from paper_2307_12059_b200 import kgc
    E, Rel = generate(800, 3, 16, seed=35)
    eps = theta_for(E, Rel, 2, 1e-2)
    with kgc.Join() as j:
        n = j.run(E, Rel, 2, eps)
        dev = torch.empty((n, 4), dtype=torch.int32, device="cuda")
        assert kgc.kgc_results(j.ctx, dev, n) == n
        host = j.results()
    got = dev.cpu().numpy()
    assert np.array_equal(got[:, :3], np.stack([host["h"], host["r"], host["t"]], 1))


# ------------------------------------------------- degenerate cases
def test_eps_zero_zero_relation_gives_self_pairs():
    E, _ = generate(500, 1, 24, seed=36, dist="uniform")
    Rel = np.zeros((3, 24), np.float32)
    for norm in (1, 2):
        res, _ = gpu_join(E, Rel, norm, 0.0)
        assert keyset(res) == {(i, r, i) for i in range(500) for r in range(3)}
        assert np.all(res["dist"] == 0)


def test_eps_huge_returns_everything():
    E, Rel = generate(150, 3, 8, seed=37)
    res, st = gpu_join(E, Rel, 2, 1e6)
    assert res.size == 150 * 150 * 3
    assert len(keyset(res)) == res.size


def test_empty_inputs():
    from paper_2307_12059_b200 import kgc
    with kgc.Join() as j:
        assert j.run(np.zeros((0, 4), np.float32), np.zeros((3, 4), np.float32), 2, 1.0) == 0
        assert j.run(np.zeros((5, 4), np.float32), np.zeros((0, 4), np.float32), 2, 1.0) == 0
        assert j.results().size == 0


def test_errors():
    from paper_2307_12059_b200 import kgc
    E, Rel = generate(64, 2, 8, seed=38)
    with kgc.Join() as j:
        bad = E.copy()
        bad[5, 3] = np.nan
        with pytest.raises(kgc.KgcError) as ei:
            j.run(bad, Rel, 2, 1.0)
        assert ei.value.status == kgc.KGC_EDATA
        badr = Rel.copy()
        badr[1, 0] = np.inf
        with pytest.raises(kgc.KgcError) as ei:
            j.run(E, badr, 2, 1.0)
        assert ei.value.status == kgc.KGC_EDATA
        for args in ((E, Rel, 3, 1.0), (E, Rel, 2, -1.0), (E, Rel, 2, float("nan"))):
            with pytest.raises(kgc.KgcError) as ei:
                j.run(*args)
            assert ei.value.status == kgc.KGC_EINVAL
        with pytest.raises(kgc.KgcError) as ei:
            kgc.kgc_results(j.ctx)
        assert ei.value.status == kgc.KGC_ESTATE
        # the context stays usable after errors
        n = j.run(E, Rel, 2, 2.0)
        assert n == j.results().size


def test_capacity_overflow_rerun():
    E, Rel = generate(600, 4, 16, seed=39)
    eps = theta_for(E, Rel, 2, 0.05)
    res, st = gpu_join(E, Rel, 2, eps, result_capacity=10)
    assert st["reruns"] >= 1
    check_parity(E, Rel, 2, eps, res)


# ------------------------------------------------- per-step checks (K1-K3)
def _quant16(keys):
    kmin, kmax = np.float32(keys.min()), np.float32(keys.max())
    rng = np.float32(kmax - kmin)
    if rng <= 0:
        return np.zeros(keys.shape, np.int64)
    x = (keys - kmin) * (np.float32(65536.0) / rng)
    return np.clip(x, 0, 65535).astype(np.int64)


@pytest.mark.parametrize("norm", [1, 2])
def test_keys_sort_ranges(norm):
    from paper_2307_12059_b200 import kgc
    E, Rel = generate(3000, 4, 40, seed=40)
    N, R = 3000, 4
    eps = theta_for(E, Rel, norm, 1e-3)
    with kgc.Join() as j:
        j.run(E, Rel, norm, eps)
        kt = j.inspect("tail_keys")
        kq = j.inspect("query_keys").reshape(R, N)
        tperm = j.inspect("tail_perm")
        qperm = j.inspect("query_perm").reshape(R, N)
        ranges = j.inspect("tile_ranges").reshape(R, -1, 2)
        st = j.stats()
    # K1: pivot distances (Dist(p, Y)) vs the oracle, FP64 rounded once to fp32
    p = np.zeros(40)
    np.testing.assert_allclose(kt, orc.pivot_distances(E, p, norm), rtol=2 ** -23, atol=0)
    for r in range(R):
        np.testing.assert_allclose(kq[r], orc.pivot_distances(orc.connector1(E, Rel[r]), p, norm), rtol=2 ** -23)
    # K2: permutations; non-decreasing 16-bit bucket; ties by ascending index (stable)
    for keys, perm in [(kt, tperm)] + [(kq[r], qperm[r]) for r in range(R)]:
        assert np.array_equal(np.sort(perm), np.arange(N))
        qk = _quant16(keys)[perm]
        assert np.all(np.diff(qk) >= 0)
        same = np.diff(qk) == 0
        assert np.all(np.diff(perm)[same] > 0)
    # K3: completeness -- every (query, tail) pair passing Lemma 1's test
    # |d(p,q) - d(p,t)| <= eps lies inside its query tile's surviving range
    BM, BN = st["query_tile_rows"], st["tail_tile_rows"]
    skt = kt[tperm]
    for r in range(R):
        skq = kq[r][qperm[r]]
        for qt in range(ranges.shape[1]):
            sb, eb = ranges[r, qt]
            rows = skq[qt * BM:(qt + 1) * BM]
            ok = np.abs(rows[:, None] - skt[None, :]) <= eps
            js = np.nonzero(ok.any(axis=0))[0] // BN
            if js.size:
                assert sb <= js.min() and js.max() <= eb


# ------------------------------------------------- full-size configs, sampled oracle
@pytest.mark.parametrize("cfg,norm,hit,S", [("c2", 2, 1e-4, 1500), ("c2", 1, 1e-4, 1500), ("c3", 2, 1e-5, 1500),
                                            ("c3", 2, 1e-3, 600), ("c4", 2, 1e-5, 300)])
def test_full_size_sampled(cfg, norm, hit, S):
    E, Rel = generate_config(cfg)
    N, R = E.shape[0], Rel.shape[0]
    rows = sample_rows(N, R, S, seed=7)
    eps = theta_for(E, Rel, norm, hit, rows=rows)
    res, st = gpu_join(E, Rel, norm, eps)
    rep = check_parity(E, Rel, norm, eps, res, rows=rows)
    assert rep["tight"] > 0
    assert st["tile_pairs_surviving"] < st["tile_pairs_total"]


# ------------------------------------------------- multi-pivot pruning (§8(f) row 2)
@pytest.mark.parametrize("K", [2, 4, 8])
@pytest.mark.parametrize("norm", [1, 2])
def test_multipivot_parity_c1(K, norm):
    E, Rel = generate_config("c1")
    eps = theta_for(E, Rel, norm, 1e-3)
    res, st = gpu_join(E, Rel, norm, eps, pivots=K)
    assert st["pivots_used"] == K
    check_parity(E, Rel, norm, eps, res)


@pytest.mark.parametrize("N,R,d", [(7, 3, 5), (300, 5, 100), (1000, 4, 200), (513, 2, 256), (700, 3, 50)])
@pytest.mark.parametrize("norm", [1, 2])
def test_multipivot_ragged(N, R, d, norm):
    E, Rel = generate(N, R, d, seed=N + 7 * d, dist="cluster")
    eps = theta_for(E, Rel, norm, 0.01)
    engines = ["tc", "simt", "tc2"] if norm == 2 else ["simt"]
    for eng in engines:
        res, st = gpu_join(E, Rel, norm, eps, pivots=8, **ENGINES[eng])
        check_parity(E, Rel, norm, eps, res)


@pytest.mark.parametrize("norm", [1, 2])
def test_multipivot_equals_single_pivot(norm):
    """Same set with 1 and 8 pivots (the tiles differ, so the surviving-tile
    counts are not ordered pair by pair; both prune)."""
    E, Rel = generate(6000, 6, 64, seed=41)
    eps = theta_for(E, Rel, norm, 1e-3)
    a, sa = gpu_join(E, Rel, norm, eps, pivots=1)
    b, sb = gpu_join(E, Rel, norm, eps, pivots=8)
    assert keyset(a) == keyset(b)
    assert sb["pivots_used"] == 8 and sa["pivots_used"] == 1
    assert sb["tile_pairs_surviving"] < sb["tile_pairs_total"]


@pytest.mark.parametrize("world", [2, 3, 8])
def test_multipivot_sharding_invariance(world):
    E, Rel = generate(3000, 7, 48, seed=42)
    eps = theta_for(E, Rel, 2, 1e-3)
    full, _ = gpu_join(E, Rel, 2, eps, pivots=8)
    parts = [gpu_join(E, Rel, 2, eps, rank=r, world=world, pivots=8)[0] for r in range(world)]
    sets = [keyset(p) for p in parts]
    assert sum(len(s) for s in sets) == len(set().union(*sets))
    assert set().union(*sets) == keyset(full)


@pytest.mark.parametrize("norm", [1, 2])
def test_multipivot_tile_lists_complete(norm):
    """Every (query, tail) pair that passes the K-pivot L_inf test of Lemma 1
    (|d(p_k,q) - d(p_k,t)| <= eps for all k) lies in a surviving tile of its
    query tile's list; keys within their documented FP32 bound of FP64."""
    from paper_2307_12059_b200 import kgc
    E, Rel = generate(2500, 3, 32, seed=43)
    N, R, K = 2500, 3, 8
    eps = theta_for(E, Rel, norm, 1e-3)
    with kgc.Join(pivots=K) as j:
        j.run(E, Rel, norm, eps)
        kt = j.inspect("tail_keys").reshape(N, K)
        kq = j.inspect("query_keys").reshape(R, N, K)
        tperm = j.inspect("tail_perm")
        qperm = j.inspect("query_perm").reshape(R, N)
        cum = j.inspect("query_cost")
        lst = j.inspect("tile_list")
        st = j.stats()
    BM, BN = st["query_tile_rows"], st["tail_tile_rows"]
    QT = st["query_tiles"]
    assert np.array_equal(np.sort(tperm), np.arange(N))
    skt = kt[tperm]
    for r in range(R):
        assert np.array_equal(np.sort(qperm[r]), np.arange(N))
        skq = kq[r][qperm[r]]
        for qt in range(QT):
            tq = r * QT + qt
            hi = cum[tq + 1] if tq + 1 < len(cum) else len(lst) + cum[0]
            tiles = set(lst[cum[tq] - cum[0]: hi - cum[0]].tolist())
            rows = skq[qt * BM:(qt + 1) * BM]
            ok = np.ones((rows.shape[0], N), bool)
            for k in range(K):
                ok &= np.abs(rows[:, None, k] - skt[None, :, k]) <= eps
            need = set((np.nonzero(ok.any(axis=0))[0] // BN).tolist())
            assert need <= tiles


@pytest.mark.parametrize("cfg,norm,hit,S", [("c2", 2, 1e-4, 1200), ("c2", 1, 1e-4, 1200), ("c3", 2, 1e-5, 800)])
def test_multipivot_full_size_sampled(cfg, norm, hit, S):
    E, Rel = generate_config(cfg)
    N, R = E.shape[0], Rel.shape[0]
    rows = sample_rows(N, R, S, seed=8)
    eps = theta_for(E, Rel, norm, hit, rows=rows)
    res, st = gpu_join(E, Rel, norm, eps, pivots=8)
    rep = check_parity(E, Rel, norm, eps, res, rows=rows)
    assert rep["tight"] > 0


# ------------------------------------------------- FP16x2 L1 engine
@pytest.mark.parametrize("eng", [1, 2])
def test_l1_engines_parity(eng):
    E, Rel = generate_config("c1")
    eps = theta_for(E, Rel, 1, 1e-3)
    res, st = gpu_join(E, Rel, 1, eps, l1_engine=eng)
    assert st["engine"] == (3 if eng == 1 else 2)
    check_parity(E, Rel, 1, eps, res)


def test_l1_half_engine_rejects_large_values():
    """|values| > 1000 leave the FP16 range margin: an explicit FP16x2 request is
    refused (EINVAL); the default engine (FP32) handles the data."""
    from paper_2307_12059_b200 import kgc
    E, Rel = generate(900, 3, 40, seed=44)
    E = (E * np.float32(3000.0)).astype(np.float32)
    Rel = (Rel * np.float32(3000.0)).astype(np.float32)
    eps = theta_for(E, Rel, 1, 1e-3)
    with pytest.raises(kgc.KgcError) as ei:
        gpu_join(E, Rel, 1, eps, l1_engine=1)
    assert ei.value.status == kgc.KGC_EINVAL
    res, st = gpu_join(E, Rel, 1, eps)
    assert st["engine"] == 2
    check_parity(E, Rel, 1, eps, res)


def test_l1_half_engine_tiny_values_and_planted_zeros():
    """Subnormal-range FP16 values and exact translations (distance 0)."""
    rng = np.random.default_rng(45)
    E = (rng.standard_normal((600, 24)) * 1e-5).astype(np.float32)
    Rel = (rng.standard_normal((3, 24)) * 1e-5).astype(np.float32)
    E[1] = E[0] + Rel[0]
    eps = theta_for(E, Rel, 1, 1e-3)
    res, st = gpu_join(E, Rel, 1, eps, l1_engine=1)
    assert st["engine"] == 3
    check_parity(E, Rel, 1, eps, res)


# ------------------------------------------------- tcgen05 on CTA pairs (l2_engine 3)
def test_tc2_engine_reported_and_tiles_256x128():
    """CTA-pair engine: 256-row query tiles (128 per CTA) x 128-row tail tiles (UMMA M = 256, N = 128)."""
    E, Rel = generate(1000, 3, 64, seed=5)
    eps = theta_for(E, Rel, 2, 1e-2)
    res, st = gpu_join(E, Rel, 2, eps, l2_engine=3)
    assert st["engine"] == 4 and st["query_tile_rows"] == 256 and st["tail_tile_rows"] == 128
    check_parity(E, Rel, 2, eps, res)


@pytest.mark.parametrize("pivots", [1, 8])
@pytest.mark.parametrize("world", [1, 3])
def test_tc2_matches_tc(pivots, world):
    """Same result set from the 1-CTA and the CTA-pair tensor-core engines, also per shard."""
    E, Rel = generate(5000, 5, 100, seed=77)
    eps = theta_for(E, Rel, 2, 1e-3, rows=sample_rows(5000, 5, 2000, seed=1))
    for r in range(world):
        a, _ = gpu_join(E, Rel, 2, eps, pivots=pivots, rank=r, world=world, l2_engine=1)
        b, sb = gpu_join(E, Rel, 2, eps, pivots=pivots, rank=r, world=world, l2_engine=3)
        assert sb["engine"] == 4
        if world == 1:
            assert keyset(a) == keyset(b)
    full_a, _ = gpu_join(E, Rel, 2, eps, pivots=pivots, l2_engine=1)
    parts = [gpu_join(E, Rel, 2, eps, pivots=pivots, rank=r, world=world, l2_engine=3)[0] for r in range(world)]
    assert set().union(*[keyset(p) for p in parts]) == keyset(full_a)


@pytest.mark.parametrize("d", [8, 200, 256])
def test_tc2_dims(d):
    """Kpad 8 (one K chunk), 200 (one A stage), 256 (largest)."""
    E, Rel = generate(900, 3, d, seed=d)
    eps = theta_for(E, Rel, 2, 1e-2)
    res, _ = gpu_join(E, Rel, 2, eps, l2_engine=3)
    check_parity(E, Rel, 2, eps, res)


@pytest.mark.parametrize("cfg,hit,S", [("c3", 1e-5, 800), ("c4", 1e-5, 300)])
def test_tc2_full_size_sampled(cfg, hit, S):
    E, Rel = generate_config(cfg)
    N, R = E.shape[0], Rel.shape[0]
    rows = sample_rows(N, R, S, seed=9)
    eps = theta_for(E, Rel, 2, hit, rows=rows)
    res, st = gpu_join(E, Rel, 2, eps, l2_engine=3, pivots=8)
    assert st["engine"] == 4
    rep = check_parity(E, Rel, 2, eps, res, rows=rows)
    assert rep["tight"] > 0


@pytest.mark.parametrize("norm,opts", [(2, dict(l2_engine=1)), (2, dict(l2_engine=3)), (2, dict(l2_engine=2)),
                                       (1, dict()), (1, dict(l1_engine=2)), (1, dict(l1_engine=1))])
@pytest.mark.parametrize("world", [2, 5])
def test_cyclic_split_invariance_multipivot(norm, opts, world):
    """split 2 (query tiles dealt round-robin to ranks): shards disjoint, union = the 1-context set,
    for every tile engine with 8 pivots (tile lists laid out over the whole query-tile range)."""
    E, Rel = generate(4000, 5, 40, seed=34)
    eps = theta_for(E, Rel, norm, 2e-3)
    full, _ = gpu_join(E, Rel, norm, eps, pivots=8, **opts)
    parts = [gpu_join(E, Rel, norm, eps, rank=r, world=world, split=2, pivots=8, **opts) for r in range(world)]
    sets = [keyset(p[0]) for p in parts]
    assert sum(len(s) for s in sets) == len(set().union(*sets))
    assert set().union(*sets) == keyset(full)
    assert sum(p[1]["tile_pairs_mine"] for p in parts) == parts[0][1]["tile_pairs_surviving"]


# ------------------------------------------------- partition-based join (§4.7)
@pytest.mark.parametrize("norm,opts", [(2, dict()), (2, dict(l2_engine=3)), (2, dict(l2_engine=2)),
                                       (2, dict(pivots=8)), (2, dict(pivots=8, l2_engine=4)), (1, dict()),
                                       (1, dict(pivots=8)), (1, dict(l1_engine=1)),
                                       # many pivots: tails from another array (own entity terms, delta_t)
                                       (2, dict(pivots=64)), (2, dict(pivots=128, l2_engine=3)),
                                       (2, dict(pivots=32, l2_engine=4)), (1, dict(pivots=32))])
@pytest.mark.parametrize("world", [2, 3])
def test_tail_partition_join(norm, opts, world):
    """tail_shard = 1: rank k joins every query against tails [kN/W, (k+1)N/W) only;
    each shard's tails lie in its partition, shards are disjoint, their union is the full set and
    matches the oracle."""
    N = 3000
    E, Rel = generate(N, 5, 40, seed=35)
    eps = theta_for(E, Rel, norm, 2e-3)
    full, _ = gpu_join(E, Rel, norm, eps, **opts)
    parts = [gpu_join(E, Rel, norm, eps, rank=r, world=world, tail_shard=1, device_inputs=(r != 1), **opts)
             for r in range(world)]
    for r, (res, st) in enumerate(parts):
        t0, t1 = N * r // world, N * (r + 1) // world
        assert np.all((res["t"] >= t0) & (res["t"] < t1)), r
        assert st["results"] == res.size
    sets = [keyset(p[0]) for p in parts]
    assert sum(len(s) for s in sets) == len(set().union(*sets))
    assert set().union(*sets) == keyset(full)
    check_parity(E, Rel, norm, eps, np.concatenate([p[0] for p in parts]))


def test_tail_partition_more_ranks_than_tails():
    E, Rel = generate(2, 3, 4, seed=36)
    eps = theta_for(E, Rel, 2, 0.3)
    full, _ = gpu_join(E, Rel, 2, eps)
    parts = [gpu_join(E, Rel, 2, eps, rank=r, world=5, tail_shard=1)[0] for r in range(5)]
    assert set().union(*[keyset(p) for p in parts]) == keyset(full)
