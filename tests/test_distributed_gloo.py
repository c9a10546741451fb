"""N > 1 host logic on CPU: two processes (gloo, world_size 2) split the query
tiles with libkgc's kgc_shard_range (the rule the device uses), each joins its
own shard, counts are all-reduced as bench.py does, and the union of the
shards equals the single-process join (sharding invariance).

The per-rank join here is the oracle restricted to the rank's query rows (no
GPU on this box); the GPU sharding itself is covered by
tests/test_gpu_parity.py::test_sharding_invariance.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

BM, BN = 128, 128


def _plan(E, Rel, norm, eps):
    """Per relation: queries sorted by pivot distance (zero pivot), query tiles of
    BM rows, surviving tail tiles by Lemma 1 at tile granularity; returns the
    sorted head order per relation and the per-query-tile surviving-tile counts."""
    from oracle import oracle
    N, R = E.shape[0], Rel.shape[0]
    p = np.zeros(E.shape[1])
    _, skt = oracle.sort_side(oracle.pivot_distances(E, p, norm))
    TT = (N + BN - 1) // BN
    tmin = np.array([skt[j * BN:(j + 1) * BN].min() for j in range(TT)])
    tmax = np.array([skt[j * BN:(j + 1) * BN].max() for j in range(TT)])
    QT = (N + BM - 1) // BM
    order, cost = [], []
    for r in range(R):
        perm, skq = oracle.sort_side(oracle.pivot_distances(oracle.connector1(E, Rel[r]), p, norm))
        order.append(perm)
        for qt in range(QT):
            rows = skq[qt * BM:(qt + 1) * BM]
            ok = (tmax >= rows.min() - eps) & (tmin <= rows.max() + eps)
            cost.append(int(ok.sum()))
    return order, np.array(cost, np.int64), QT


def _worker(rank, world, port, E, Rel, norm, eps, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2307_12059_b200 import kgc
        N, R = E.shape[0], Rel.shape[0]
        order, cost, QT = _plan(E, Rel, norm, eps)
        cum = np.concatenate([[0], np.cumsum(cost)[:-1]])
        total = int(cost.sum())
        b, e, my_cost = kgc.kgc_shard_range(cum, total, rank, world)
        rows = []
        for tq in range(b, e):
            r, qt = divmod(tq, QT)
            for h in order[r][qt * BM:(qt + 1) * BM]:
                rows.append(int(h) * R + r)
        res = oracle.join(E, Rel, norm, eps, rows=np.sort(np.array(rows, np.int64))) if rows else \
            np.zeros(0, oracle.TRIPLET_DTYPE)
        counts = torch.tensor([res.size, my_cost], dtype=torch.int64)
        dist.all_reduce(counts)                      # as bench.py does after every step
        gathered = [None] * world
        dist.all_gather_object(gathered, (b, e, [tuple(x) for x in zip(res["h"], res["r"], res["t"])]))
        # the library's multi-GPU finish: count all-gather + results gathered to rank 0
        res16 = np.zeros(res.size, kgc.TRIPLET_DTYPE)
        for f in ("h", "r", "t"):
            res16[f] = res[f]
        res16["dist"] = res["dist"].astype(np.float32)
        cnts, allres = kgc.gather_results(res16, root=0)
        assert sum(cnts) == int(counts[0]) and cnts[rank] == res.size
        if rank == 0:
            q.put((int(counts[0]), int(counts[1]), total, gathered, allres))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("norm", [1, 2])
def test_two_rank_shards_union_equals_full_join(norm):
    from oracle import oracle
    from synth import generate
    E, Rel = generate(700, 5, 16, seed=50)
    D = np.sort(oracle.dist_rows(E, Rel, norm).ravel())
    eps = float(np.float32(0.5 * (D[2000] + D[2001])))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, E, Rel, norm, eps, q)) for r in range(2)]
    for p in procs:
        p.start()
    n_all, cost_all, total, gathered, allres = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = oracle.join(E, Rel, norm, eps)
    full_set = set(zip(full["h"].tolist(), full["r"].tolist(), full["t"].tolist()))
    shards = [set(g[2]) for g in gathered]
    assert not (shards[0] & shards[1])
    assert shards[0] | shards[1] == full_set
    assert n_all == len(full_set)
    # gather_results: rank 0 holds every shard's records, in rank order, nothing lost or duplicated
    assert allres.size == n_all
    assert set(zip(allres["h"].tolist(), allres["r"].tolist(), allres["t"].tolist())) == full_set
    assert cost_all == total
    (b0, e0, _), (b1, e1, _) = gathered
    assert b0 == 0 and e0 == b1          # contiguous split of the query tiles


# ------------------------------------------------ partition-based ring join (host logic)
def _ring_worker(rank, world, port, E, Rel, norm, eps, bounds, q):
    """kgc.partition_join over gloo with libkgc's block join replaced, in this test process
    only, by an oracle block join: exercises the ring (block sizes / offsets exchange, send /
    recv order, which block each step holds) without a GPU."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import oracle
        from paper_2307_12059_b200 import kgc
        state = {}

        class _Ctx:
            def _follow_torch_stream(self, x):
                pass

            def close(self):
                pass

            ctx = None

        def block(ctx, Eh, Nh, h_off, Et, Nt, t_off, Rel_, R, d, norm_, eps_):
            Eh, Et = np.asarray(Eh), np.asarray(Et)
            Ecat = np.vstack([Eh, Et])
            rows = (np.arange(Nh)[:, None] * R + np.arange(R)[None, :]).ravel()
            res = oracle.join(Ecat, np.asarray(Rel_), norm_, eps_, rows=rows)
            res = res[res["t"] >= Nh]
            out = np.zeros(res.size, kgc.TRIPLET_DTYPE)
            out["h"], out["r"], out["t"] = res["h"] + h_off, res["r"], res["t"] - Nh + t_off
            out["dist"] = res["dist"]
            state["res"] = out
            state.setdefault("blocks", []).append((h_off, t_off, Nt))

        def results(ctx, out=None, capacity=None):
            r = state["res"]
            if out is not None:
                out.numpy().reshape(-1).view(kgc.TRIPLET_DTYPE)[:r.size] = r
            return r.size

        kgc.kgc_join_block = block
        kgc.kgc_results = results
        a, b = bounds[rank]
        mine = kgc.partition_join(torch.from_numpy(E[a:b].copy()), a, Rel, norm, eps, join=_Ctx())
        recs = mine.numpy().reshape(-1).view(kgc.TRIPLET_DTYPE)
        q.put((rank, [tuple(x) for x in zip(recs["h"].tolist(), recs["r"].tolist(), recs["t"].tolist())],
               state.get("blocks", [])))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_partition_ring_covers_every_block_pair_once(world):
    from oracle import oracle
    from synth import generate
    E, Rel = generate(301, 3, 12, seed=51)
    norm = 2
    D = np.sort(oracle.dist_rows(E, Rel, norm).ravel())
    eps = float(np.float32(0.5 * (D[900] + D[901])))
    cuts = [0, 90, 200, 301][:world] + [301] if world == 3 else [0, 130, 301]
    bounds = [(cuts[i], cuts[i + 1]) for i in range(world)]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ring_worker, args=(r, world, port, E, Rel, norm, eps, bounds, q))
             for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = oracle.join(E, Rel, norm, eps)
    full_set = set(zip(full["h"].tolist(), full["r"].tolist(), full["t"].tolist()))
    sets = {r: set(s) for r, s, _ in got}
    assert sum(len(s) for s in sets.values()) == len(set().union(*sets.values()))   # disjoint
    assert set().union(*sets.values()) == full_set
    for r, _, blocks in got:
        a, b = bounds[r]
        assert all(h_off == a for h_off, _, _ in blocks)
        assert sorted(t for _, t, _ in blocks) == sorted(x[0] for x in bounds)     # every tail block once
        for res_h in sets[r]:
            assert a <= res_h[0] < b
