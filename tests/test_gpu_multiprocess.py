"""Multi-process paths on the one B200 (gloo process group, two or three processes on
cuda:0): real libkgc shards, not oracle stand-ins.

  * query-tile shards (kgc_options rank / world, tails replicated) joined in separate
    processes, results collected with kgc.gather_results, union vs the oracle;
  * the partition-based ring join (kgc.partition_join, §4.7): every
    process holds one entity block, tail blocks pass around the ring, union vs the oracle.

NCCL cannot put two ranks on one GPU, so the ring's transport here is gloo over host
tensors; on a multi-GPU node the same code moves device tensors with NCCL send / recv.
"""
import os
import socket

import numpy as np
import pytest

from synth import generate
from tests.gpu_util import check_parity, theta_for

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2307_12059_b200 import _build
    _build.build()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, mode, E, Rel, norm, eps, opts, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2307_12059_b200 import kgc
        torch.cuda.set_device(0)
        N = E.shape[0]
        Rt = torch.from_numpy(Rel).cuda()
        if mode == "shards":
            Et = torch.from_numpy(E).cuda()
            with kgc.Join(rank=rank, world=world, **opts) as j:
                j.run(Et, Rt, norm, eps)
                mine = j.results()
            counts, allres = kgc.gather_results(mine, root=0)
            info = {"results": mine.size}
        else:
            a, b = N * rank // world, N * (rank + 1) // world
            Eb = torch.from_numpy(E[a:b].copy()).cuda()
            recs = kgc.partition_join(Eb, a, Rt, norm, eps, **opts)
            mine = recs.cpu().numpy().reshape(-1).view(kgc.TRIPLET_DTYPE)
            assert np.all((mine["h"] >= a) & (mine["h"] < b))
            counts, allres = kgc.gather_results(mine, root=0)
            info = {"results": mine.size, "resident_input_floats": int((b - a) * E.shape[1] * 3)}
        if rank == 0:
            q.put((counts, allres, info))
    finally:
        dist.destroy_process_group()


def _run(world, mode, E, Rel, norm, eps, **opts):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, E, Rel, norm, eps, opts, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("norm,opts", [(2, dict()), (2, dict(pivots=8)), (1, dict(pivots=8)), (2, dict(split=2)),
                                       (2, dict(tail_shard=1)), (2, dict(pivots=96)), (2, dict(pivots=64, tail_shard=1)),
                                       (2, dict(split=3, pivots=96)), (1, dict(split=3, pivots=8))])
def test_two_process_shards_gathered(norm, opts):
    E, Rel = generate(3000, 5, 40, seed=81)
    eps = theta_for(E, Rel, norm, 2e-3)
    counts, allres, _ = _run(2, "shards", E, Rel, norm, eps, **opts)
    assert allres.size == sum(counts)
    check_parity(E, Rel, norm, eps, allres)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("norm,opts", [(2, dict()), (2, dict(pivots=8)), (1, dict(pivots=8)), (2, dict(l2_engine=3)),
                                       (2, dict(pivots=64))])
def test_partition_ring_join(world, norm, opts):
    N = 4000
    E, Rel = generate(N, 5, 48, seed=82 + world)
    eps = theta_for(E, Rel, norm, 2e-3)
    counts, allres, info = _run(world, "ring", E, Rel, norm, eps, **opts)
    assert allres.size == sum(counts)
    check_parity(E, Rel, norm, eps, allres)
    # per-process resident inputs: own block + two tail buffers = 3 N d / W floats
    assert info["resident_input_floats"] <= 3 * (N // world + 1) * E.shape[1]
