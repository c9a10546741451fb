"""The C-ABI library loads and exports every symbol include/kgc.h declares;
host-only logic (no GPU needed)."""
import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def lib():
    from paper_2307_12059_b200 import _build
    _build.build()
    from paper_2307_12059_b200 import kgc
    return kgc.load_library()


def _header_functions():
    src = (ROOT / "include" / "kgc.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(kgc_[a-z_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _header_functions()
    for n in ("kgc_create", "kgc_join", "kgc_results", "kgc_stats", "kgc_last_error", "kgc_destroy"):
        assert n in names


def test_library_exports_every_declared_symbol(lib):
    for name in _header_functions():
        assert hasattr(lib, name), name
    from paper_2307_12059_b200 import kgc
    assert sorted(kgc.EXPORTS) == _header_functions()


def test_abi_version(lib):
    assert lib.kgc_abi_version() == 3


def test_struct_sizes_match_header():
    from paper_2307_12059_b200 import kgc
    assert kgc.TRIPLET_DTYPE.itemsize == 16
    assert ctypes.sizeof(kgc.kgc_options) == 64  # relation_batch fills the tail padding
    # kgc_stats_t: compile a tiny C program against the header to get its size
    import subprocess
    import tempfile
    with tempfile.TemporaryDirectory() as td:
        c = Path(td) / "s.c"
        c.write_text('#include "kgc.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                     'int main(){printf("%zu %zu %zu\\n", sizeof(kgc_stats_t), sizeof(kgc_options), '
                     'offsetof(kgc_stats_t, ms_recheck));return 0;}\n')
        exe = Path(td) / "s"
        subprocess.check_call(["gcc", f"-I{ROOT / 'include'}", str(c), "-o", str(exe)])
        a, b, off = map(int, subprocess.check_output([str(exe)]).split())
    assert a == ctypes.sizeof(kgc.kgc_stats_t)
    assert b == ctypes.sizeof(kgc.kgc_options)
    assert off == kgc.kgc_stats_t.ms_recheck.offset


def test_default_options():
    from paper_2307_12059_b200 import kgc
    o = kgc.kgc_default_options()
    assert (o.device, o.rank, o.world, o.prune, o.pivot, o.l2_engine) == (-1, 0, 1, 1, 0, 0)
    assert o.result_capacity == 0 and not o.stream


def test_create_without_gpu_fails_loudly():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2307_12059_b200 import kgc
    with pytest.raises(kgc.KgcError) as ei:
        kgc.kgc_create()
    assert ei.value.status in (kgc.KGC_ENODEV, kgc.KGC_ECUDA)


def test_invalid_options_rejected():
    from paper_2307_12059_b200 import kgc
    with pytest.raises(kgc.KgcError) as ei:
        kgc.kgc_create(world=2, rank=2)
    assert ei.value.status == kgc.KGC_EINVAL


def _shard_reference(cum, total, world):
    """The documented rule (include/kgc.h): owner(q) = min(W-1, floor(W cum[q] / total))."""
    if total == 0:
        return np.zeros(len(cum), dtype=np.int64)
    return np.minimum(world - 1, (world * np.asarray(cum, np.int64)) // total)


@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_range_partitions_and_balances(world):
    from paper_2307_12059_b200 import kgc
    rng = np.random.default_rng(world)
    cost = rng.integers(0, 50, size=1000)
    cost[rng.random(1000) < 0.3] = 0
    cum = np.concatenate([[0], np.cumsum(cost)[:-1]])
    total = int(cost.sum())
    owner = _shard_reference(cum, total, world)
    covered = []
    costs = []
    for rank in range(world):
        b, e, c = kgc.kgc_shard_range(cum, total, rank, world)
        assert np.all(owner[b:e] == rank)
        assert c == int(cost[b:e].sum())
        covered.append((b, e))
        costs.append(c)
    # contiguous, disjoint, covering [0, n)
    nonempty = [x for x in covered if x[1] > x[0]]
    assert nonempty[0][0] == 0 and nonempty[-1][1] == 1000
    for (b0, e0), (b1, e1) in zip(nonempty, nonempty[1:]):
        assert e0 == b1
    assert sum(costs) == total
    assert max(costs) <= total / world + cost.max()


def test_shard_range_rejects_bad_args():
    from paper_2307_12059_b200 import kgc
    with pytest.raises(kgc.KgcError):
        kgc.kgc_shard_range([0, 1], 2, 3, 2)


@pytest.mark.parametrize("N,world,chunk", [(0, 3, 4096), (1, 1, 4096), (5, 8, 4096), (2500, 4, 4096),
                                           (14951, 8, 4096), (123182, 8, 4096), (1000000, 8, 4096),
                                           (1000000, 3, 1000), (77777, 5, 8192)])
def test_spatial_chunks_partition(N, world, chunk):
    """split = 3 host rule (include/kgc.h): over all ranks the chunks partition [0, N) exactly,
    every rank owns m or fewer chunks dealt c mod world, chunk sizes differ by at most one, and
    every rank's head count is within one chunk of N / world."""
    from paper_2307_12059_b200 import kgc
    seen = np.zeros(N, dtype=np.int64)
    heads = []
    sizes = []
    for rank in range(world):
        b, ln = kgc.kgc_spatial_chunks(N, world, rank, chunk)
        for x, y in zip(b, ln):
            assert y >= 1
            seen[x:x + y] += 1
            sizes.append(int(y))
        if len(b) > 1:
            assert np.all(np.diff(b) > 0)          # chunk order
        heads.append(int(ln.sum()))
    assert np.all(seen == 1)                        # exact partition
    if sizes:
        assert max(sizes) - min(sizes) <= 1
        assert max(heads) - min(heads) <= max(sizes)
        m = max(2, round(N / (world * chunk)))
        assert len(sizes) == min(N, world * m)


def test_spatial_chunks_rejects_bad_args():
    from paper_2307_12059_b200 import kgc
    for args in [(-1, 2, 0), (10, 0, 0), (10, 2, 2), (10, 2, -1)]:
        with pytest.raises(kgc.KgcError):
            kgc.kgc_spatial_chunks(*args)
    with pytest.raises(kgc.KgcError):
        kgc.kgc_spatial_chunks(10, 2, 0, chunk=0)
