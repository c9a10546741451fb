"""Thin ctypes binding of libkgc (include/kgc.h) -- argument marshalling only.

Every step of the join runs in the CUDA kernels of libkgc.so; this module
only converts Python / numpy / torch arguments into pointers and sizes.
There is no fallback: if libkgc.so is missing or cannot be loaded, importing
the library raises.

Same names as the C ABI: kgc_default_options, kgc_create, kgc_join,
kgc_results, kgc_stats, kgc_last_error, kgc_set_stream, kgc_destroy,
kgc_inspect, kgc_shard_range, kgc_topk, kgc_join_se, kgc_join_block,
kgc_abi_version.  ``Join`` is a small convenience wrapper around one context;
``gather_results`` and ``partition_join`` are the multi-GPU plumbing over a
torch process group (bytes only: every step of the method runs in libkgc).
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import numpy as np

LIB_PATH = Path(__file__).resolve().parent / "libkgc.so"

KGC_OK, KGC_EINVAL, KGC_EDATA, KGC_ENOMEM, KGC_ECUDA, KGC_ENODEV, KGC_ESTATE = 0, -1, -2, -3, -4, -5, -6
STATUS_NAMES = {0: "KGC_OK", -1: "KGC_EINVAL", -2: "KGC_EDATA", -3: "KGC_ENOMEM", -4: "KGC_ECUDA",
                -5: "KGC_ENODEV", -6: "KGC_ESTATE"}
KGC_MAX_DIM = 1024
INSPECT = {"tail_keys": 1, "query_keys": 2, "tail_perm": 3, "query_perm": 4, "tile_ranges": 5, "query_cost": 6,
           "tile_list": 7, "gather_list": 8, "gather_cost": 9, "pivots": 10}

TRIPLET_DTYPE = np.dtype([("h", np.int32), ("r", np.int32), ("t", np.int32), ("dist", np.float32)])


class kgc_options(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("prune", ctypes.c_int32), ("pivot", ctypes.c_int32), ("l2_engine", ctypes.c_int32),
                ("chunk_tiles", ctypes.c_int32), ("pivots", ctypes.c_int32),
                ("result_capacity", ctypes.c_int64), ("stream", ctypes.c_void_p), ("l1_engine", ctypes.c_int32),
                ("split", ctypes.c_int32), ("tail_shard", ctypes.c_int32), ("relation_batch", ctypes.c_int32)]


class kgc_stats_t(ctypes.Structure):
    _fields_ = [("N", ctypes.c_int64), ("R", ctypes.c_int64), ("d", ctypes.c_int32), ("norm", ctypes.c_int32),
                ("eps", ctypes.c_float), ("rank", ctypes.c_int32), ("world", ctypes.c_int32),
                ("triplets", ctypes.c_double), ("query_tile_rows", ctypes.c_int64),
                ("tail_tile_rows", ctypes.c_int64), ("query_tiles", ctypes.c_int64), ("tail_tiles", ctypes.c_int64),
                ("tile_pairs_total", ctypes.c_int64), ("tile_pairs_surviving", ctypes.c_int64),
                ("tile_pairs_mine", ctypes.c_int64), ("work_items_mine", ctypes.c_int64),
                ("candidates", ctypes.c_int64), ("results", ctypes.c_int64), ("h2d_bytes", ctypes.c_int64),
                ("d2h_bytes", ctypes.c_int64), ("launches", ctypes.c_int32), ("reruns", ctypes.c_int32),
                ("ms_total", ctypes.c_float), ("ms_h2d", ctypes.c_float), ("ms_keys", ctypes.c_float),
                ("ms_sort", ctypes.c_float), ("ms_ranges", ctypes.c_float), ("ms_stage", ctypes.c_float),
                ("ms_tiles", ctypes.c_float), ("ms_recheck", ctypes.c_float), ("pivots_used", ctypes.c_int32),
                ("engine", ctypes.c_int32), ("ms_split", ctypes.c_float), ("ms_host", ctypes.c_float),
                ("gathered_pairs", ctypes.c_int64)]

    def as_dict(self):
        return {name: getattr(self, name) for name, _ in self._fields_}


EXPORTS = ["kgc_abi_version", "kgc_default_options", "kgc_create", "kgc_join", "kgc_results", "kgc_stats",
           "kgc_last_error", "kgc_set_stream", "kgc_destroy", "kgc_inspect", "kgc_shard_range", "kgc_topk",
           "kgc_join_se", "kgc_join_block", "kgc_spatial_chunks"]

_lib = None


def load_library(path: str | Path | None = None):
    """Load libkgc.so (raises OSError if it is missing: no fallback path exists)."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else LIB_PATH
    if not p.exists():
        raise OSError(f"libkgc.so not found at {p}; build it with `python -m paper_2307_12059_b200._build`")
    L = ctypes.CDLL(str(p))
    vp, i32, i64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    L.kgc_abi_version.restype = ctypes.c_int
    L.kgc_default_options.argtypes = [ctypes.POINTER(kgc_options)]
    L.kgc_default_options.restype = None
    L.kgc_create.argtypes = [ctypes.POINTER(vp), ctypes.POINTER(kgc_options)]
    L.kgc_create.restype = ctypes.c_int
    L.kgc_join.argtypes = [vp, vp, vp, i64, i64, i32, i32, ctypes.c_float]
    L.kgc_join.restype = ctypes.c_int
    L.kgc_results.argtypes = [vp, vp, i64]
    L.kgc_results.restype = i64
    L.kgc_stats.argtypes = [vp, ctypes.POINTER(kgc_stats_t)]
    L.kgc_stats.restype = ctypes.c_int
    L.kgc_last_error.argtypes = [vp]
    L.kgc_last_error.restype = ctypes.c_char_p
    L.kgc_set_stream.argtypes = [vp, vp]
    L.kgc_set_stream.restype = ctypes.c_int
    L.kgc_destroy.argtypes = [vp]
    L.kgc_destroy.restype = None
    L.kgc_inspect.argtypes = [vp, i32, vp, i64]
    L.kgc_inspect.restype = i64
    L.kgc_shard_range.argtypes = [vp, i64, i64, i32, i32, ctypes.POINTER(i64), ctypes.POINTER(i64)]
    L.kgc_shard_range.restype = i64
    L.kgc_spatial_chunks.argtypes = [i64, i32, i32, i64, vp, vp, i64]
    L.kgc_spatial_chunks.restype = i64
    L.kgc_topk.argtypes = [vp, vp, vp, i64, i64, i32, i32, i64, i32, vp]
    L.kgc_topk.restype = i64
    L.kgc_join_se.argtypes = [vp, vp, vp, vp, i64, i64, i32, ctypes.c_float]
    L.kgc_join_se.restype = ctypes.c_int
    L.kgc_join_block.argtypes = [vp, vp, i64, i64, vp, i64, i64, vp, i64, i32, i32, ctypes.c_float]
    L.kgc_join_block.restype = ctypes.c_int
    if path is None:
        _lib = L
    return L


class KgcError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


# ----------------------------------------------------------- raw C names

def kgc_abi_version() -> int:
    return load_library().kgc_abi_version()


def kgc_default_options(**overrides) -> kgc_options:
    o = kgc_options()
    load_library().kgc_default_options(ctypes.byref(o))
    for k, v in overrides.items():
        setattr(o, k, v)
    return o


def kgc_last_error(ctx=None) -> str:
    s = load_library().kgc_last_error(ctx)
    return s.decode() if s else ""


def kgc_create(options: kgc_options | None = None, **overrides):
    o = options if options is not None else kgc_default_options(**overrides)
    ctx = ctypes.c_void_p()
    rc = load_library().kgc_create(ctypes.byref(ctx), ctypes.byref(o))
    if rc != KGC_OK:
        raise KgcError(rc, kgc_last_error(None))
    return ctx


def _ptr(x):
    """Pointer of a numpy array or torch tensor (host or device), contiguous float32/int."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):          # torch tensor
        if not x.is_contiguous():
            raise ValueError("tensor must be contiguous")
        return ctypes.c_void_p(x.data_ptr())
    if isinstance(x, np.ndarray):
        if not x.flags["C_CONTIGUOUS"]:
            raise ValueError("array must be C-contiguous")
        return ctypes.c_void_p(x.ctypes.data)
    if isinstance(x, int):
        return ctypes.c_void_p(x)
    raise TypeError(f"unsupported buffer type {type(x)}")


def _check_f32(x, name):
    dt = getattr(x, "dtype", None)
    if dt is None:
        return
    if str(dt) not in ("float32", "torch.float32"):
        raise TypeError(f"{name} must be float32, got {dt}")


def kgc_join(ctx, E, Rel, N: int, R: int, d: int, norm: int, eps: float) -> None:
    _check_f32(E, "E")
    _check_f32(Rel, "Rel")
    rc = load_library().kgc_join(ctx, _ptr(E), _ptr(Rel), int(N), int(R), int(d), int(norm), float(eps))
    if rc != KGC_OK:
        raise KgcError(rc, kgc_last_error(ctx))


def kgc_results(ctx, out=None, capacity: int | None = None) -> int:
    cap = 0 if out is None else (capacity if capacity is not None else
                                 (out.shape[0] if hasattr(out, "shape") else 0))
    n = load_library().kgc_results(ctx, _ptr(out), int(cap))
    if n < 0:
        raise KgcError(int(n), kgc_last_error(ctx))
    return int(n)


def kgc_stats(ctx) -> dict:
    st = kgc_stats_t()
    rc = load_library().kgc_stats(ctx, ctypes.byref(st))
    if rc != KGC_OK:
        raise KgcError(rc, kgc_last_error(ctx))
    return st.as_dict()


def kgc_set_stream(ctx, stream) -> None:
    ptr = stream if isinstance(stream, int) or stream is None else getattr(stream, "cuda_stream", stream)
    rc = load_library().kgc_set_stream(ctx, ctypes.c_void_p(ptr) if ptr else None)
    if rc != KGC_OK:
        raise KgcError(rc, kgc_last_error(ctx))


def kgc_destroy(ctx) -> None:
    if ctx:
        load_library().kgc_destroy(ctx)


def kgc_inspect(ctx, what: str) -> np.ndarray:
    code = INSPECT[what]
    n = load_library().kgc_inspect(ctx, code, None, 0)
    if n < 0:
        raise KgcError(int(n), kgc_last_error(ctx))
    dtype = {"tail_keys": np.float32, "query_keys": np.float32, "tail_perm": np.int32, "query_perm": np.int32,
             "tile_ranges": np.int32, "query_cost": np.int64, "tile_list": np.int32, "gather_list": np.int32,
             "gather_cost": np.int64, "pivots": np.float32}[what]
    out = np.empty(n // np.dtype(dtype).itemsize, dtype=dtype)
    rc = load_library().kgc_inspect(ctx, code, out.ctypes.data, n)
    if rc < 0:
        raise KgcError(int(rc), kgc_last_error(ctx))
    return out


def kgc_shard_range(cum, total: int, rank: int, world: int):
    """Pure host function: the query-tile shard [begin, end) of `rank` and its cost."""
    cum = np.ascontiguousarray(cum, dtype=np.int64)
    b, e = ctypes.c_int64(), ctypes.c_int64()
    cost = load_library().kgc_shard_range(cum.ctypes.data, cum.shape[0], int(total), int(rank), int(world),
                                          ctypes.byref(b), ctypes.byref(e))
    if cost < 0:
        raise KgcError(int(cost), "kgc_shard_range: invalid argument")
    return int(b.value), int(e.value), int(cost)


def kgc_spatial_chunks(N: int, world: int, rank: int, chunk: int = 4096):
    """Pure host function (split = 3): the (begin, len) chunks of the curve order that `rank` joins."""
    L = load_library()
    n = L.kgc_spatial_chunks(int(N), int(world), int(rank), int(chunk), None, None, 0)
    if n < 0:
        raise KgcError(int(n), "kgc_spatial_chunks: invalid argument")
    b, ln = np.zeros(max(n, 1), dtype=np.int64), np.zeros(max(n, 1), dtype=np.int64)
    L.kgc_spatial_chunks(int(N), int(world), int(rank), int(chunk), b.ctypes.data, ln.ctypes.data, n)
    return b[:n], ln[:n]


def kgc_topk(ctx, E, Rel, N: int, R: int, d: int, norm: int, k: int, exclude_self: bool = False, out=None):
    """The k smallest distances over all triplets (see include/kgc.h); returns a
    TRIPLET_DTYPE array (or fills `out`, host array or device tensor, and returns the count)."""
    _check_f32(E, "E")
    _check_f32(Rel, "Rel")
    buf = out if out is not None else np.empty(max(int(k), 1), dtype=TRIPLET_DTYPE)
    n = load_library().kgc_topk(ctx, _ptr(E), _ptr(Rel), int(N), int(R), int(d), int(norm), int(k),
                                int(bool(exclude_self)), _ptr(buf))
    if n < 0:
        raise KgcError(int(n), kgc_last_error(ctx))
    return int(n) if out is not None else buf[:n]


def kgc_join_se(ctx, E, Wl, Wr, N: int, R: int, d: int, eps: float) -> None:
    """Structured Embedding join (see include/kgc.h); results via kgc_results."""
    for x, n in ((E, "E"), (Wl, "Wl"), (Wr, "Wr")):
        _check_f32(x, n)
    rc = load_library().kgc_join_se(ctx, _ptr(E), _ptr(Wl), _ptr(Wr), int(N), int(R), int(d), float(eps))
    if rc != KGC_OK:
        raise KgcError(rc, kgc_last_error(ctx))


def kgc_join_block(ctx, Eh, Nh: int, h_off: int, Et, Nt: int, t_off: int, Rel, R: int, d: int, norm: int,
                   eps: float) -> None:
    """One head block x tail block of the partition-based join (see include/kgc.h)."""
    for x, n in ((Eh, "Eh"), (Et, "Et"), (Rel, "Rel")):
        _check_f32(x, n)
    rc = load_library().kgc_join_block(ctx, _ptr(Eh), int(Nh), int(h_off), _ptr(Et), int(Nt), int(t_off), _ptr(Rel),
                                       int(R), int(d), int(norm), float(eps))
    if rc != KGC_OK:
        raise KgcError(rc, kgc_last_error(ctx))


# ----------------------------------------------------------- multi-GPU finish

def gather_results(res, root: int = 0, group=None):
    """Multi-GPU finish: all-gather of the per-rank result
    counts, then the sharded (h, r, t, dist) lists gathered to `root` by
    point-to-point transfers over the process group (NCCL for device tensors,
    gloo for host arrays).  Plumbing only: no arithmetic of the method.

    `res`: this rank's results, a TRIPLET_DTYPE numpy array or an (n, 4)
    int32 torch tensor holding the same 16-byte records (host or device).
    Returns (counts, gathered): the per-rank counts (every rank) and, on
    `root`, the concatenation in rank order as a TRIPLET_DTYPE array (None
    elsewhere)."""
    import torch
    import torch.distributed as dist
    if isinstance(res, np.ndarray):
        t = torch.from_numpy(np.ascontiguousarray(res).view(np.int32).reshape(-1, 4))
    else:
        t = res.reshape(-1, 4).contiguous()
    if dist.get_backend(group) == "nccl" and t.device.type != "cuda":
        t = t.cuda()
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    cnt = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(cnt, n, group=group)
    counts = [int(c.item()) for c in cnt]
    if rank != root:
        if counts[rank]:
            dist.send(t, dist.get_global_rank(group, root) if group is not None else root, group=group)
        return counts, None
    parts = []
    for src in range(world):
        if src == root:
            parts.append(t)
        elif counts[src]:
            buf = torch.empty((counts[src], 4), dtype=torch.int32, device=t.device)
            dist.recv(buf, dist.get_global_rank(group, src) if group is not None else src, group=group)
            parts.append(buf)
    allr = torch.cat(parts) if parts else torch.empty((0, 4), dtype=torch.int32)
    return counts, allr.cpu().numpy().reshape(-1).view(TRIPLET_DTYPE)


def partition_join(E_local, h_off: int, Rel, norm: int, eps: float, group=None, join=None, **options):
    """Partition-based join over a process group (§4.7).

    Rank k holds only entity block k: E_local = rows [h_off, h_off + n_k) of E (blocks may
    differ in size).  The tail blocks travel around a ring of ranks: at step s rank k holds
    block (k - s) mod W, joins its own heads against it with kgc_join_block (every tcgen05 /
    SIMT step of the hot path runs in libkgc) while the block is forwarded to rank k + 1 and
    the next one received from rank k - 1 (NCCL send/recv of device tensors, overlapped with
    the join; gloo with host tensors), so after W steps every (head block, tail block) pair
    has been joined exactly once and the union over ranks is R(eps).  Per-GPU resident
    inputs: the own block plus two tail buffers -- 3 N d / W floats instead of N d.

    Returns this rank's records (h, r, t global) as an (n, 4) int32 tensor on the join's
    device (TRIPLET_DTYPE records; kgc.gather_results collects them).  `join`: an existing
    kgc.Join to use (world 1), else one is created with **options.  Plumbing only: the ring
    moves bytes, libkgc computes."""
    import torch
    import torch.distributed as dist
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    nccl = dist.get_backend(group) == "nccl"
    dev = E_local.device if hasattr(E_local, "device") else torch.device("cpu")
    comm_dev = dev if nccl else torch.device("cpu")
    Eh = E_local if hasattr(E_local, "data_ptr") else torch.from_numpy(np.ascontiguousarray(E_local))
    n, d = int(Eh.shape[0]), int(Eh.shape[1])
    R = int(Rel.shape[0])
    meta = torch.tensor([n, int(h_off)], dtype=torch.int64, device=comm_dev)
    allm = [torch.zeros_like(meta) for _ in range(world)]
    dist.all_gather(allm, meta, group=group)
    sizes = [int(m[0]) for m in allm]
    offs = [int(m[1]) for m in allm]
    cap = max(sizes) if sizes else 0
    gr = (lambda r: dist.get_global_rank(group, r)) if group is not None else (lambda r: r)
    bufs = [torch.empty((max(cap, 1), d), dtype=torch.float32, device=comm_dev) for _ in range(2)]
    bufs[0][:n].copy_(Eh.to(comm_dev))
    own = join is None
    j = join if join is not None else Join(**options)
    out = []
    try:
        cur = 0
        for step in range(world):
            src = (rank - step) % world  # owner of the tail block held now
            works = []
            if step + 1 < world:
                ops = [dist.P2POp(dist.isend, bufs[cur], gr((rank + 1) % world), group),
                       dist.P2POp(dist.irecv, bufs[1 - cur], gr((rank - 1) % world), group)]
                works = dist.batch_isend_irecv(ops)
            tails = bufs[cur][:sizes[src]]
            if sizes[src] and n and R:
                j._follow_torch_stream(tails)
                kgc_join_block(j.ctx, Eh, n, int(h_off), tails, sizes[src], offs[src], Rel, R, d, norm, eps)
                cnt = kgc_results(j.ctx)
                part = torch.empty((cnt, 4), dtype=torch.int32, device=dev)
                if cnt:
                    kgc_results(j.ctx, part, cnt)
                out.append(part)
            for w in works:
                w.wait()
            cur = 1 - cur
    finally:
        if own:
            j.close()
    return torch.cat(out) if out else torch.empty((0, 4), dtype=torch.int32, device=dev)


# ----------------------------------------------------------- convenience

class Join:
    """One libkgc context.  ``run(E, Rel, norm, eps)`` joins and returns the
    result count; ``results()`` returns a numpy structured array (h, r, t, dist)."""

    def __init__(self, **options):
        stream = options.pop("stream", None)
        self.ctx = kgc_create(**options)
        self._own_order = stream is None
        if stream is not None:
            kgc_set_stream(self.ctx, stream)

    def _follow_torch_stream(self, x):
        """Without an explicit stream, a join on CUDA tensors runs on torch's current
        stream of their device, so it is ordered after the kernels that produced them
        (include/kgc.h, "Stream order")."""
        if self._own_order and getattr(x, "is_cuda", False):
            import torch
            kgc_set_stream(self.ctx, torch.cuda.current_stream(x.device).cuda_stream)

    def run(self, E, Rel, norm: int, eps: float) -> int:
        N, d = (int(E.shape[0]), int(E.shape[1])) if E is not None and len(E.shape) == 2 else (0, 1)
        R = int(Rel.shape[0]) if Rel is not None else 0
        if Rel is not None and len(Rel.shape) == 2 and R and int(Rel.shape[1]) != d:
            raise ValueError("E and Rel dimensions differ")
        self._follow_torch_stream(E)
        kgc_join(self.ctx, E, Rel, N, R, d, norm, eps)
        return kgc_results(self.ctx)

    def results(self, out=None):
        n = kgc_results(self.ctx)
        if out is None:
            out = np.empty(n, dtype=TRIPLET_DTYPE)
        kgc_results(self.ctx, out, n)
        return out

    def stats(self) -> dict:
        return kgc_stats(self.ctx)

    def run_se(self, E, Wl, Wr, eps: float) -> int:
        N, d = int(E.shape[0]), int(E.shape[1])
        self._follow_torch_stream(E)
        kgc_join_se(self.ctx, E, Wl, Wr, N, int(Wl.shape[0]), d, eps)
        return kgc_results(self.ctx)

    def run_block(self, Eh, h_off: int, Et, t_off: int, Rel, norm: int, eps: float) -> int:
        """kgc_join_block: heads Eh (global rows h_off..) against tails Et (global rows t_off..)."""
        d = int(Eh.shape[1])
        self._follow_torch_stream(Eh)
        kgc_join_block(self.ctx, Eh, int(Eh.shape[0]), h_off, Et, int(Et.shape[0]), t_off, Rel, int(Rel.shape[0]), d,
                       norm, eps)
        return kgc_results(self.ctx)

    def topk(self, E, Rel, norm: int, k: int, exclude_self: bool = False):
        N, d = int(E.shape[0]), int(E.shape[1])
        self._follow_torch_stream(E)
        return kgc_topk(self.ctx, E, Rel, N, int(Rel.shape[0]), d, norm, k, exclude_self)

    def inspect(self, what: str) -> np.ndarray:
        return kgc_inspect(self.ctx, what)

    def close(self):
        if self.ctx:
            kgc_destroy(self.ctx)
            self.ctx = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
