"""One shard of a W-rank join on one GPU (diagnostic; for ncu launch lists of the split paths).
usage: python scripts/shard_once.py c4 8 3 [rank]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2307_12059_b200 import kgc  # noqa: E402
from synth import generate_config  # noqa: E402

cfg, W, split = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
rank = int(sys.argv[4]) if len(sys.argv) > 4 else 0
thr = bench.load_thresholds()
hit = bench.DEFAULT_HIT[cfg]
eps = float(thr[cfg][f"L2@{hit:g}"]["theta"])
E, Rel = generate_config(cfg)
Et, Rt = torch.from_numpy(E).cuda(), torch.from_numpy(Rel).cuda()
with kgc.Join(device=0, rank=rank, world=W, split=split, pivots=bench.BEST_PIVOTS[cfg]) as j:
    for _ in range(2):
        j.run(Et, Rt, 2, eps)
    torch.cuda.synchronize()
    print(json.dumps({k: v for k, v in j.stats().items() if k.startswith("ms_")}))
