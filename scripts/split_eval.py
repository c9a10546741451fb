"""Offline check of split estimators against per-relation ground truth (CPU, diagnostic).

Reads the JSON lines of scripts/relation_costs.py, regenerates the seeded inputs,
computes candidate per-relation cost estimates in numpy, and simulates the
rank-local split (contiguous query-tile ranges by cumulative estimated cost,
uniform within a relation) at W = 2, 4, 8: reported is max over ranks of the
TRUE cost / (total / W).

usage: python scripts/split_eval.py gpurun_out/relation_costs.jsonl
"""
from __future__ import annotations

import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from synth import generate_config  # noqa: E402


def simulate(est, true, W):
    R = len(est)
    cum = np.concatenate([[0.0], np.cumsum(est)])
    total = cum[-1]
    cuts = [0.0]
    for k in range(1, W):
        t = total * k / W
        r = int(np.searchsorted(cum, t, side="right") - 1)
        r = min(r, R - 1)
        frac = (t - cum[r]) / est[r]
        cuts.append(r + frac)
    cuts.append(float(R))
    # true cost of fractional relation range [a, b)
    tcum = np.concatenate([[0.0], np.cumsum(true)])

    def at(x):
        r = min(int(x), R - 1)
        return tcum[r] + (x - r) * true[r]
    loads = [at(cuts[k + 1]) - at(cuts[k]) for k in range(W)]
    return max(loads) / (tcum[-1] / W)


def main():
    for line in open(sys.argv[1]):
        d = json.loads(line)
        name, eps = d["config"], d["eps"]
        rel = d["relations"]
        true = np.array([r["ms_tiles"] + r["ms_recheck"] + 0.02 for r in rel])
        pairs = np.array([r["tile_pairs_surviving"] for r in rel], float)
        E, Rel = generate_config(name)
        N, dd = E.shape
        R = Rel.shape[0]
        ests = {"uniform": np.ones(R), "oracle_pairs": pairs + 1}
        # current: zero-pivot element count |‖q‖ - ‖t‖| <= theta
        S = 256
        heads = (np.arange(S) * N // S)
        kt = np.sort(np.linalg.norm(E.astype(np.float64), axis=1))
        cur = np.zeros(R)
        for r in range(R):
            kq = np.linalg.norm(E[heads].astype(np.float64) + Rel[r], axis=1)
            cur[r] = (np.searchsorted(kt, kq + eps, "right") - np.searchsorted(kt, kq - eps, "left")).sum() + 1
        ests["current_1pivot"] = cur
        # sampled density: ||q - t|| <= rho for T evenly spaced tails
        for T in (1024, 4096):
            for Sq in (64, 256):
                tails = E[(np.arange(T) * N // T)].astype(np.float64)
                tn = (tails ** 2).sum(1)
                hs = (np.arange(Sq) * N // Sq)
                D = []
                for r in range(R):
                    q = E[hs].astype(np.float64) + Rel[r]
                    D.append((q ** 2).sum(1)[:, None] + tn[None, :] - 2 * q @ tails.T)
                D = np.sqrt(np.maximum(np.stack(D), 0))  # R x Sq x T
                for m in (2, 4, 8, 16):
                    c = (D <= m * eps).sum((1, 2)) + 1.0
                    ests[f"dens_T{T}_S{Sq}_x{m}"] = c
                flat = np.sort(D.ravel())
                for f in (1e-4, 1e-3, 1e-2):
                    rho = flat[int(f * flat.size)]
                    ests[f"dens_T{T}_S{Sq}_q{f:g}"] = (D <= rho).sum((1, 2)) + 1.0
        print(f"== {name}: R={R}, true cost total {true.sum():.1f} ms, "
              f"cv {true.std() / true.mean():.2f}, pairs corr with ms {np.corrcoef(pairs, true)[0, 1]:.3f}")
        for k, e in ests.items():
            cc = np.corrcoef(np.log(e), np.log(true))[0, 1] if e.std() > 0 else 0.0
            print(f"  {k:28s} logcorr {cc:6.3f}  W2 {simulate(e, true, 2):.3f}  W4 {simulate(e, true, 4):.3f}  "
                  f"W8 {simulate(e, true, 8):.3f}")


if __name__ == "__main__":
    main()
