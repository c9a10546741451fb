"""Time kgc_join_se (SE) on an SE-shaped synthetic config (device inputs,
CUDA events).  usage (under gpurun): python scripts/bench_se.py [N R d hit]"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2307_12059_b200 import kgc  # noqa: E402
from synth import generate_se  # noqa: E402

N, R, d = (int(x) for x in sys.argv[1:4]) if len(sys.argv) >= 4 else (40943, 18, 100)
hit = float(sys.argv[4]) if len(sys.argv) >= 5 else 1e-4
E, Wl, Wr = generate_se(N, R, d, seed=2)
# theta from FP64 connectors of 64 sampled heads of relation 0 against all tails (test-side
# calibration only; the join itself never sees these values)
E64 = E.astype(np.float64)
A = E64[:64] @ Wl[0].astype(np.float64).T
B = E64 @ Wr[0].astype(np.float64).T
D = np.sort(np.abs(A[:, None, :] - B[None, :, :]).sum(axis=2).ravel())
k = max(1, int(hit * D.size))
eps = float(np.float32(0.5 * (D[k] + D[k + 1])))
args = [torch.from_numpy(x).cuda() for x in (E, Wl, Wr)]
s = torch.cuda.current_stream()
with kgc.Join(stream=s.cuda_stream) as j:
    j.run_se(*args, eps)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    n = j.run_se(*args, eps)
    b.record(s)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    st = j.stats()
print(json.dumps({"model": "SE", "N": N, "R": R, "d": d, "eps": eps, "hit_rate_target": hit, "ms": ms,
                  "candidate_triplets_per_s": N * N * R / (ms / 1e3), "results": n,
                  "pruned_tile_fraction": 1 - st["tile_pairs_surviving"] / max(1, st["tile_pairs_total"]),
                  "ms_tiles": st["ms_tiles"], "ms_recheck": st["ms_recheck"], "ms_keys": st["ms_keys"]}))
