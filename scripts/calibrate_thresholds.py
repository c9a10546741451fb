"""Write configs/thresholds.json: theta per (config, norm, hit rate).

Calls only oracle/ (FP64 distances of a seeded row sample, SURVEY.md §8(d)
"theta calibration"; reading R14) and synth/ (inputs).  bench.py
reads the committed file; it never calibrates itself.

usage: python scripts/calibrate_thresholds.py [c1 c2 ...]
"""
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle  # noqa: E402
from synth import CONFIGS, GENERATOR_VERSION, generate_config, sample_rows  # noqa: E402

PLAN = {
    "c1": {2: [1e-3], 1: [1e-3]},
    "c2": {2: [1e-5, 1e-4, 1e-3], 1: [1e-5, 1e-4, 1e-3]},
    "c3": {2: [1e-6, 1e-5, 1e-4, 1e-3]},
    "c4": {2: [1e-6, 1e-5, 1e-4]},
    "c5": {2: [1e-8, 1e-7, 1e-6]},
}
SAMPLE = {"c1": None, "c2": 4096, "c3": 4096, "c4": 2048, "c5": 100}


def main(names):
    out_path = ROOT / "configs" / "thresholds.json"
    data = json.loads(out_path.read_text()) if out_path.exists() else {}
    data["_about"] = ("theta (distance threshold, float32-exact) per config / norm / target hit rate, calibrated by "
                      "scripts/calibrate_thresholds.py with oracle.calibrate_theta: the midpoint of the k-th and "
                      "(k+1)-th smallest FP64 dist3 over a seeded row sample (k = hit rate x sample size), moved "
                      "below any self-edge distance ||r_j||_p within 2e-4*theta (DESIGN.md reading R14), rounded to "
                      "float32.")
    data["generator"] = GENERATOR_VERSION
    for name in names:
        c = CONFIGS[name]
        E, Rel = generate_config(name)
        S = SAMPLE[name]
        rows = sample_rows(c.N, c.R, S, seed=c.seed) if S else None
        if rows is None:
            import numpy as np
            rows = np.arange(c.N * c.R)
        entry = data.setdefault(name, {"N": c.N, "R": c.R, "d": c.d, "seed": c.seed, "sample_rows": int(len(rows))})
        for norm, hits in PLAN[name].items():
            for hit in hits:
                t0 = time.time()
                theta, info = oracle.calibrate_theta(E, Rel, norm, hit, rows)
                entry[f"L{norm}@{hit:g}"] = {"theta": theta, **info}
                print(f"{name} L{norm} hit {hit:g}: theta={theta!r} sample hit rate {info['hit_rate_sample']:.3g} "
                      f"({time.time() - t0:.1f}s)", flush=True)
        out_path.write_text(json.dumps(data, indent=1, sort_keys=True))


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3", "c4"])
