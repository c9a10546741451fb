"""How many pivots? (diagnostic).  Runs one K = 8 join (libkgc), takes its sort orders (Hilbert
code of the first 4 pivots) and pivots, extends the farthest-point traversal to 32 pivots in numpy
on the library's sample, and counts the (query tile x tail tile) pairs that survive the L_inf test
of mp_survives with the first K pivots, K = 4 ... 32, for 256 x 128 tiles (the pair engine).
usage: python scripts/pivot_sweep.py c4 1e-5"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2307_12059_b200 import kgc  # noqa: E402
from synth import generate_config  # noqa: E402

name, hit = sys.argv[1], float(sys.argv[2])
KMAX = int(sys.argv[3]) if len(sys.argv) > 3 else 32
th = json.loads((ROOT / "configs" / "thresholds.json").read_text())[name][f"L2@{hit:g}"]["theta"]
E, Rel = generate_config(name)
N, R, d = E.shape[0], Rel.shape[0], E.shape[1]
with kgc.Join(pivots=8, l2_engine=3) as j:
    j.run(torch.from_numpy(E).cuda(), torch.from_numpy(Rel).cuda(), 2, th)
    st = j.stats()
    P8 = j.inspect("pivots").reshape(8, d).astype(np.float64)
    tperm = j.inspect("tail_perm")
    qperm = j.inspect("query_perm").reshape(R, N)
E64 = torch.from_numpy(E).cuda().double()
R64 = torch.from_numpy(Rel).cuda().double()
# continue the farthest-point traversal on the library's sample (rows s N / S)
S = min(1024, (200 * 1024 // 4 - d) // (d | 1), N)
X = E64[torch.arange(S, device="cuda") * N // S]
P = [torch.from_numpy(p).cuda() for p in P8]
mind = torch.stack([((X - p) ** 2).sum(1) for p in P]).min(0).values
while len(P) < KMAX:
    i = int(torch.argmax(mind))
    P.append(X[i].clone())
    mind = torch.minimum(mind, ((X - X[i]) ** 2).sum(1))
Pm = torch.stack(P)                                   # [16, d]
A = ((E64[:, None, :] - Pm[None]) ** 2).sum(2)        # [N, 16] ||h - p||^2
kt = A.sqrt()
HR = E64 @ R64.T                                      # [N, R]
C = R64 @ Pm.T                                        # [R, 16]
rr = (R64 ** 2).sum(1)
relm = (d + 8) * 2.0 ** -23
BQ, BT = 256, 128


def boxes(sk, rows):
    n = sk.shape[0]
    nt = (n + rows - 1) // rows
    pad = nt * rows - n
    a = torch.cat([sk, sk[-1:].expand(pad, -1)]) if pad else sk
    a = a.reshape(nt, rows, -1)
    return a.min(1).values, a.max(1).values


tp = torch.from_numpy(tperm.astype(np.int64)).cuda()
tmn, tmx = boxes(kt[tp], BT)
out = {"config": name, "hit": hit, "lib_tile_pairs": st["tile_pairs_surviving"], "tiles": f"{BQ}x{BT}"}
Ks = [k for k in (4, 8, 12, 16, 20, 24, 32, 40, 48, 64, 96, 128) if k <= KMAX]
surv = {K: 0 for K in Ks}
for r in range(R):
    kq = (A + 2 * HR[:, r:r + 1] - 2 * C[r][None] + rr[r]).clamp_min(0).sqrt()  # [N, 16]
    qp = torch.from_numpy(qperm[r].astype(np.int64)).cuda()
    qmn, qmx = boxes(kq[qp], BQ)
    ok = torch.ones((qmn.shape[0], tmn.shape[0]), dtype=torch.bool, device="cuda")
    for k in range(KMAX):
        thk = th * (1 + 2 ** -14) + relm * (qmx[:, None, k].abs() + tmx[None, :, k].abs())
        ok &= ~((tmx[None, :, k] < qmn[:, None, k] - thk) | (tmn[None, :, k] > qmx[:, None, k] + thk))
        if k + 1 in surv:
            surv[k + 1] += int(ok.sum())
for K in Ks:
    out[f"K{K}"] = {"tile_pairs": surv[K], "pair_frac": surv[K] * BQ * BT / (N * N * R)}
print(json.dumps(out), flush=True)
