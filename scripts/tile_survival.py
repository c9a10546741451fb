"""Tile-pair survival of the K-pivot L_inf test for other tile shapes (diagnostic).

Runs one join, reads the K-pivot keys and sort orders libkgc computed (kgc_inspect), and counts
surviving (query tile, tail tile) pairs and the pairs they contain for several tile heights with the
same test and margin as mp_survives (pivots.cu).  usage: python scripts/tile_survival.py c4 1e-5"""
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
th = json.loads((ROOT / "configs" / "thresholds.json").read_text())[name][f"L2@{hit:g}"]["theta"]
E, Rel = generate_config(name)
N, R, d = E.shape[0], Rel.shape[0], E.shape[1]
K = 8
with kgc.Join(pivots=K, l2_engine=3) as j:
    j.run(torch.from_numpy(E).cuda(), torch.from_numpy(Rel).cuda(), 2, th)
    st = j.stats()
    kt = j.inspect("tail_keys").reshape(N, K)
    kq = j.inspect("query_keys").reshape(R, N, K)
    tperm = j.inspect("tail_perm")
    qperm = j.inspect("query_perm").reshape(R, N)
relm = (d + 8) * 2.0 ** -23
qn_marg = 0.0  # the query-box widening (2^-23 max||q||) is negligible here


def boxes(sk, rows):
    n = sk.shape[0]
    nt = (n + rows - 1) // rows
    pad = nt * rows - n
    a = np.concatenate([sk, np.repeat(sk[-1:], pad, 0)]) if pad else sk
    a = a.reshape(nt, rows, K)
    return a.min(1), a.max(1)


skt = kt[tperm]
out = {"config": name, "lib_tile_pairs_surviving": st["tile_pairs_surviving"], "lib_tile_rows": [st["query_tile_rows"],
                                                                                                    st["tail_tile_rows"]]}
for bq, bn in [(256, 256), (256, 128), (256, 64), (128, 256), (128, 128)]:
    tmn, tmx = boxes(skt, bn)
    surv_tiles = 0
    for r in range(R):
        skq = kq[r][qperm[r]]
        qmn, qmx = boxes(skq, bq)
        ok = np.ones((qmn.shape[0], tmn.shape[0]), bool)
        for k in range(K):
            thk = th * (1 + 2 ** -14) + relm * (np.abs(qmx[:, None, k]) + np.abs(tmx[None, :, k]))
            ok &= ~((tmx[None, :, k] < qmn[:, None, k] - thk) | (tmn[None, :, k] > qmx[:, None, k] + thk))
        surv_tiles += int(ok.sum())
    out[f"{bq}x{bn}"] = {"tile_pairs": surv_tiles, "pair_frac": surv_tiles * bq * bn / (N * N * R)}
    print(json.dumps(out), flush=True)
