"""GPU: the spatial block-cyclic head split (kgc_options.split = 3, csrc/split.cu; SURVEY §8(e),
PAPER.md:156 "a block which can be processed in parallel").  Every rank orders the heads along
the same space-filling curve and joins the heads of its chunks against all tails: the shards
must be disjoint, their union the one-context set, and that set must match the oracle
(Definition 1)."""
import numpy as np
import pytest

from synth import generate, generate_config, sample_rows
from tests.gpu_util import check_parity, gpu_join, keyset, theta_for

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2307_12059_b200 import _build
    _build.build()


def _shards(E, Rel, norm, eps, world, **opts):
    return [gpu_join(E, Rel, norm, eps, rank=r, world=world, split=3, **opts) for r in range(world)]


def _sorted_keys(res):
    k = np.stack([res["h"].astype(np.int64), res["r"].astype(np.int64), res["t"].astype(np.int64)], 1)
    return k[np.lexsort((k[:, 2], k[:, 1], k[:, 0]))]


@pytest.mark.parametrize("norm,opts", [(2, dict()), (2, dict(pivots=8)), (2, dict(pivots=64)),
                                       (2, dict(pivots=96, l2_engine=3)), (2, dict(l2_engine=2)),
                                       (1, dict()), (1, dict(pivots=8)), (1, dict(pivots=32))])
@pytest.mark.parametrize("world", [2, 3, 8])
def test_spatial_split_union_is_oracle_set(norm, opts, world):
    E, Rel = generate(3000, 6, 40, seed=91)
    eps = theta_for(E, Rel, norm, 2e-3)
    full, sf = gpu_join(E, Rel, norm, eps, **opts)
    parts = _shards(E, Rel, norm, eps, world, **opts)
    sets = [keyset(p[0]) for p in parts]
    assert sum(len(s) for s in sets) == len(set().union(*sets))      # disjoint
    assert set().union(*sets) == keyset(full)
    union = np.concatenate([p[0] for p in parts])
    check_parity(E, Rel, norm, eps, union)
    for r, (_, st) in enumerate(parts):
        assert st["rank"] == r and st["world"] == world
        assert st["N"] == 3000 and st["triplets"] == sf["triplets"]


def test_spatial_split_heads_partition():
    """Every head appears in exactly one shard (self pairs at r = 0 mark each head's owner)."""
    E, Rel = generate(2500, 3, 24, seed=92)
    Rel[0] = 0.0                                                  # (h, 0, h) at distance 0 for every h
    eps = theta_for(E, Rel, 2, 1e-3)
    owners = np.full(2500, -1)
    for r, (res, _) in enumerate(_shards(E, Rel, 2, eps, 4)):
        self_pairs = res[(res["r"] == 0) & (res["h"] == res["t"])]["h"]
        assert (owners[self_pairs] == -1).all()
        owners[self_pairs] = r
    assert (owners >= 0).all()
    counts = np.bincount(owners, minlength=4)
    assert counts.max() - counts.min() <= 2                        # W * m equal chunks (+-1 head each)


@pytest.mark.parametrize("N,world", [(5, 8), (9, 4), (257, 3), (1031, 5)])
def test_spatial_split_ragged_and_tiny(N, world):
    """N below the chunk count (ranks without heads return 0 results) and ragged chunk sizes."""
    E, Rel = generate(N, 4, 20, seed=93 + N)
    eps = theta_for(E, Rel, 2, 5e-2)
    full, _ = gpu_join(E, Rel, 2, eps)
    parts = _shards(E, Rel, 2, eps, world)
    sets = [keyset(p[0]) for p in parts]
    assert sum(len(s) for s in sets) == len(set().union(*sets))
    assert set().union(*sets) == keyset(full)


def test_spatial_split_host_inputs():
    E, Rel = generate(2000, 5, 32, seed=94)
    eps = theta_for(E, Rel, 2, 2e-3)
    full, _ = gpu_join(E, Rel, 2, eps, pivots=8)
    parts = [gpu_join(E, Rel, 2, eps, device_inputs=False, rank=r, world=3, split=3, pivots=8) for r in range(3)]
    sets = [keyset(p[0]) for p in parts]
    assert sum(len(s) for s in sets) == len(set().union(*sets)) == len(keyset(full))
    assert all(p[1]["h2d_bytes"] >= E.nbytes for p in parts)


@pytest.mark.parametrize("K", [8, 64])
def test_spatial_split_relation_batches(K):
    E, Rel = generate(3000, 7, 40, seed=95)
    eps = theta_for(E, Rel, 2, 2e-3)
    full, _ = gpu_join(E, Rel, 2, eps, pivots=K)
    parts = _shards(E, Rel, 2, eps, 3, pivots=K, relation_batch=2)
    sets = [keyset(p[0]) for p in parts]
    assert sum(len(s) for s in sets) == len(set().union(*sets))
    assert set().union(*sets) == keyset(full)


@pytest.mark.parametrize("cfg,K", [("c4", 96), ("c3", 64)])
def test_spatial_split_full_size(cfg, K):
    """BASELINE configs at full size, 8 shards in the bench's launch configuration: the union equals
    the one-GPU set record for record; 300 sampled query rows against the oracle."""
    import json
    from pathlib import Path
    E, Rel = generate_config(cfg)
    thr = json.loads((Path(__file__).resolve().parents[1] / "configs" / "thresholds.json").read_text())
    eps = float(thr[cfg]["L2@1e-05"]["theta"])
    full, _ = gpu_join(E, Rel, 2, eps, pivots=K)
    parts = _shards(E, Rel, 2, eps, 8, pivots=K)
    union = np.concatenate([p[0] for p in parts])
    assert union.size == full.size
    assert np.array_equal(_sorted_keys(union), _sorted_keys(full))
    rows = sample_rows(E.shape[0], Rel.shape[0], 300, seed=96)
    check_parity(E, Rel, 2, eps, union, rows=rows)


def test_c5_eight_shards_full_size():
    """The north star's 8-GPU configuration as bench.py launches it (c5: 1M entities, R = 100,
    d = 128, L2, 128 pivots, split 3, W = 8), each shard in turn on the one GPU: the shards' counts
    add up to the one-GPU join's, and 100 uniformly sampled (h, r) rows plus 100 rows with hits are
    checked over all 10^6 tails against the oracle (no missing, extra or duplicate triplet)."""
    import json
    from pathlib import Path

    import torch

    from paper_2307_12059_b200 import kgc
    E, Rel = generate_config("c5")
    N, R = E.shape[0], Rel.shape[0]
    thr = json.loads((Path(__file__).resolve().parents[1] / "configs" / "thresholds.json").read_text())
    eps = float(thr["c5"]["L2@1e-06"]["theta"])
    Et, Rt = torch.from_numpy(E).cuda(), torch.from_numpy(Rel).cuda()
    with kgc.Join(pivots=128) as j:
        j.run(Et, Rt, 2, eps)
        n_full = kgc.kgc_results(j.ctx)
        t = torch.empty((n_full, 4), dtype=torch.int32, device="cuda")
        kgc.kgc_results(j.ctx, t, n_full)
        keys = np.unique((t[:, 0].long() * R + t[:, 1].long()).cpu().numpy())
        del t
    rng = np.random.default_rng(19)
    rows = np.union1d(sample_rows(N, R, 100, seed=18), rng.choice(keys, min(100, keys.size), replace=False))
    rows_t = torch.from_numpy(rows.astype(np.int64)).cuda()
    parts, n_sum = [], 0
    for rank in range(8):
        with kgc.Join(pivots=128, rank=rank, world=8, split=3) as j:
            j.run(Et, Rt, 2, eps)
            n = kgc.kgc_results(j.ctx)
            n_sum += n
            t = torch.empty((max(n, 1), 4), dtype=torch.int32, device="cuda")
            kgc.kgc_results(j.ctx, t, n)
            t = t[:n]
            m = torch.isin(t[:, 0].long() * R + t[:, 1].long(), rows_t)
            parts.append(np.ascontiguousarray(t[m].cpu().numpy()).reshape(-1).view(kgc.TRIPLET_DTYPE))
    assert n_sum == n_full and n_full > 10 ** 7
    got = np.concatenate(parts)
    rep = check_parity(E, Rel, 2, eps, got, rows=rows)
    assert rep["tight"] > 50, rep
