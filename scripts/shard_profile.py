"""One shard of a W-rank join, repeated (diagnostic for per-rank fixed costs under ncu).

usage: python scripts/shard_profile.py c3 8 [rank] [split] [pivots]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2307_12059_b200 import kgc  # noqa: E402
from synth import generate_config  # noqa: E402

name, W = sys.argv[1], int(sys.argv[2])
rank = int(sys.argv[3]) if len(sys.argv) > 3 else 0
split = int(sys.argv[4]) if len(sys.argv) > 4 else 0
pivots = int(sys.argv[5]) if len(sys.argv) > 5 else {"c3": 1}.get(name, 8)
hit = {"c3": 1e-5, "c4": 1e-5, "c5": 1e-6, "c2": 1e-4}[name]
th = json.loads((ROOT / "configs" / "thresholds.json").read_text())[name][f"L2@{hit:g}"]["theta"]
E, Rel = generate_config(name)
Et, Rt = torch.from_numpy(E).cuda(), torch.from_numpy(Rel).cuda()
with kgc.Join(rank=rank, world=W, split=split, pivots=pivots) as j:
    for _ in range(3):
        j.run(Et, Rt, 2, th)
    st = j.stats()
print(json.dumps({k: round(v, 4) if isinstance(v, float) else v for k, v in st.items()}))
