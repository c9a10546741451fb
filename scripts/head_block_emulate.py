"""Projected W-GPU step of the head-block split (diagnostic, one GPU).

Rank k of W joins the heads [kN/W, (k+1)N/W) of every relation against all N
tails (kgc_join_block with the tails replicated): the query side -- keys, sort,
tile test, tiles, re-check -- is split by heads, so no rank preprocesses
another's queries and no cost estimate is needed; heads are spread over the
embedding space, so every rank sees a similar mix of dense and empty query
regions.  Every shard runs in turn on one GPU (CUDA events, L2 flushed before
each); max over shards projects the W-GPU device time.  The result counts of
the shards must add up to the full join's.

usage: python scripts/head_block_emulate.py c5 c4 c3 > gpurun_out/head_block.jsonl
"""
from __future__ import annotations

import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_12059_b200 import kgc  # noqa: E402
from synth import generate_config  # noqa: E402

KEYS = ("tile_pairs_mine", "candidates", "results", "ms_keys", "ms_sort", "ms_ranges", "ms_tiles", "ms_recheck",
        "ms_total")


def timed(fn, stream, flush, steps):
    fn()
    ts = []
    for _ in range(steps):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.mean(ts)


def main():
    thr = bench.load_thresholds()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    args = [a for a in sys.argv[1:] if not a.startswith("--")] or ["c5"]
    steps = 3
    spatial = "--spatial" in sys.argv or "--cyclic" in sys.argv
    plan = [(2, 0), (4, 0), (8, 0)]
    if "--cyclic" in sys.argv:
        plan = [(8, 1024), (8, 4096), (8, 16384), (2, 4096), (4, 4096)]
    for name in args:
        hit = bench.DEFAULT_HIT[name]
        piv = bench.BEST_PIVOTS[name]
        eps = float(thr[name][f"L2@{hit:g}"]["theta"])
        E, Rel = generate_config(name)
        Et, Rt = torch.from_numpy(E).to(dev), torch.from_numpy(Rel).to(dev)
        N = E.shape[0]
        with kgc.Join(device=0, pivots=piv, stream=stream.cuda_stream) as j:
            full_ms = timed(lambda: j.run(Et, Rt, 2, eps), stream, flush, steps)
            full_n = kgc.kgc_results(j.ctx)
            tperm = torch.from_numpy(j.inspect("tail_perm").astype("int64")).to(dev)
        order = tperm if spatial else torch.arange(N, device=dev)
        for W, C in plan:
            shard_ms, phases, total_n = [], [], 0
            for k in range(W):
                h0, h1 = N * k // W, N * (k + 1) // W
                if C:  # block-cyclic over the spatial order: chunks k, k + W, k + 2W, ...
                    idx = torch.cat([order[c:c + C] for c in range(k * C, N, W * C)])
                else:
                    idx = order[h0:h1]
                Eh = Et[idx].contiguous()
                if spatial:
                    h0 = 0
                with kgc.Join(device=0, pivots=piv, stream=stream.cuda_stream) as j:
                    shard_ms.append(timed(lambda: j.run_block(Eh, h0, Et, 0, Rt, 2, eps), stream, flush, steps))
                    st = j.stats()
                    total_n += kgc.kgc_results(j.ctx)
                phases.append({k2: round(st[k2], 3) if isinstance(st[k2], float) else st[k2] for k2 in KEYS})
            ms = max(shard_ms)
            print(json.dumps({"config": name, "split": "spatial-head-block" if spatial else "head-block", "W": W, "chunk": C, "pivots": piv, "full_ms": full_ms,
                              "shard_ms": shard_ms, "projected_ms": ms,
                              "efficiency": full_ms / (W * ms), "results_full": full_n, "results_shards": total_n,
                              "phases": phases}), flush=True)


if __name__ == "__main__":
    main()
