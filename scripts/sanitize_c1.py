"""Run every tile engine once on c1 (N=1000, R=10, d=50) -- the workload for the
compute-sanitizer passes (memcheck / racecheck / synccheck) committed under profiles/.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_c1.py [--quick]
Checks each result set against the oracle, so a sanitizer run that perturbed nothing still
proves the engines it exercised are the ones the parity tests cover."""
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle  # noqa: E402
from paper_2307_12059_b200 import kgc  # noqa: E402
from synth import generate_config  # noqa: E402

RUNS = [(2, dict(l2_engine=1)), (2, dict(l2_engine=2)), (2, dict(l2_engine=3)), (2, dict(l2_engine=1, pivots=8)),
        (2, dict(l2_engine=3, pivots=8)), (2, dict(l2_engine=4, pivots=8)), (2, dict(l2_engine=5)),
        (2, dict(l2_engine=6, pivots=8)), (1, dict(l1_engine=2)), (1, dict(l1_engine=3, pivots=8)),
        (1, dict(l1_engine=1)), (1, dict(l1_engine=2, pivots=8)),
        # round 2: many pivots (FP64-factorised L2 keys, on-the-fly boxes, staged tile test, one-CTA sorts)
        (2, dict(l2_engine=1, pivots=64)), (2, dict(l2_engine=3, pivots=64)), (2, dict(l2_engine=4, pivots=32)),
        (1, dict(l1_engine=3, pivots=32))]


def main():
    E, Rel = generate_config("c1")
    rows = np.arange(E.shape[0] * Rel.shape[0])
    Et, Rt = torch.from_numpy(E).cuda(), torch.from_numpy(Rel).cuda()
    runs = RUNS[:3] if "--quick" in sys.argv else RUNS
    for norm, opts in runs:
        eps, _ = oracle.calibrate_theta(E, Rel, norm, 1e-3, rows)
        with kgc.Join(**opts) as j:
            j.run(Et, Rt, norm, eps)
            res = j.results()
            st = j.stats()
        rep = oracle.compare(res, oracle.join(E, Rel, norm, eps * (1 + 1e-4)), eps)
        print(f"L{norm} {opts}: engine {st['engine']}, {res.size} triplets, parity {rep['ok']}", flush=True)
        assert rep["ok"], rep


if __name__ == "__main__":
    main()
