"""Relation-factored L2 (l2_engine 5) against the per-relation tensor-core
engine on one config and distribution (device inputs, CUDA events, median of 5 joins).
usage (under gpurun): python scripts/bench_factored.py [config dist hit]"""
import json
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402  (test-side theta calibration only)
from paper_2307_12059_b200 import kgc  # noqa: E402
from synth import CONFIGS, generate, sample_rows  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
dist = sys.argv[2] if len(sys.argv) > 2 else "uniform"
hit = float(sys.argv[3]) if len(sys.argv) > 3 else 1e-5
c = CONFIGS[cfg]
E, Rel = generate(c.N, c.R, c.d, seed=c.seed, dist=dist)
rows = sample_rows(c.N, c.R, 512, seed=12)
eps, _ = oracle.calibrate_theta(E, Rel, 2, hit, rows)
Et, Rt = torch.from_numpy(E).cuda(), torch.from_numpy(Rel).cuda()
s = torch.cuda.current_stream()
out = {"config": cfg, "dist": dist, "hit": hit, "eps": eps}
for name, opts in (("per_relation", dict(l2_engine=1)), ("per_relation_k8", dict(l2_engine=1, pivots=8)),
                   ("factored", dict(l2_engine=5))):
    with kgc.Join(stream=s.cuda_stream, **opts) as j:
        j.run(Et, Rt, 2, eps)
        ts = []
        for _ in range(5):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            n = j.run(Et, Rt, 2, eps)
            b.record(s)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        st = j.stats()
    ms = statistics.median(ts)
    out[name] = {"ms": ms, "triplets_per_s": c.N * c.N * c.R / (ms / 1e3), "results": n,
                 "pruned_tile_fraction": 1 - st["tile_pairs_surviving"] / max(1, st["tile_pairs_total"]),
                 "ms_tiles": st["ms_tiles"], "ms_recheck": st["ms_recheck"], "candidates": st["candidates"]}
print(json.dumps(out))
