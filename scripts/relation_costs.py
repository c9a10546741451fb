"""Per-relation ground truth for the multi-GPU split estimate (diagnostic, GPU).

Joins every relation of a config on its own (one relation per kgc_join, the
config's pivots and theta) and records the surviving tile pairs, candidates and
device phase times.  Pivots are chosen from the tails alone, so each relation's
query tiles see the same tail boxes as in the full join: these are the costs a
rank-local split should balance.  Output: one JSON line per config.

usage: python scripts/relation_costs.py c5 c4 c3 > gpurun_out/relation_costs.jsonl
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_12059_b200 import kgc  # noqa: E402
from synth import generate_config  # noqa: E402


def main():
    thr = bench.load_thresholds()
    dev = torch.device("cuda", 0)
    for name in sys.argv[1:] or ["c5"]:
        hit = bench.DEFAULT_HIT[name]
        piv = bench.BEST_PIVOTS[name]
        eps = float(thr[name][f"L2@{hit:g}"]["theta"])
        E, Rel = generate_config(name)
        Et, Rt = torch.from_numpy(E).to(dev), torch.from_numpy(Rel).to(dev)
        R = Rel.shape[0]
        rows = []
        with kgc.Join(device=0, pivots=piv) as j:
            j.run(Et, Rt[0:1].contiguous(), 2, eps)  # warm-up
            for r in range(R):
                j.run(Et, Rt[r:r + 1].contiguous(), 2, eps)
                st = j.stats()
                rows.append({k: (round(v, 4) if isinstance(v, float) else v) for k, v in st.items()
                             if k in ("tile_pairs_surviving", "tile_pairs_mine", "work_items_mine", "candidates",
                                      "results", "ms_total", "ms_keys", "ms_sort", "ms_ranges", "ms_tiles",
                                      "ms_recheck")})
        print(json.dumps({"config": name, "hit": hit, "pivots": piv, "eps": eps, "relations": rows}), flush=True)


if __name__ == "__main__":
    main()
