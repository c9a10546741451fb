"""A/B timing of libkgc engine options on one workload (diagnostic, not the bench line).

usage: python scripts/engine_ab.py c4 2 1e-5 'pivots=8' 'pivots=8,l2_engine=4' ...
Prints, per option set, the mean per-phase device times (libkgc's CUDA events) over
--steps joins after --warmup, the surviving / gathered pair fractions and the result count.
"""
import json
import statistics
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2307_12059_b200 import kgc  # noqa: E402
from synth import generate_config  # noqa: E402


def parse(s):
    out = {}
    for kv in filter(None, s.split(",")):
        k, v = kv.split("=")
        out[k] = int(v)
    return out


def main():
    name, norm, hit = sys.argv[1], int(sys.argv[2]), float(sys.argv[3])
    steps = 5
    th = json.loads((ROOT / "configs" / "thresholds.json").read_text())[name][f"L{norm}@{hit:g}"]["theta"]
    E, Rel = generate_config(name)
    N, R = E.shape[0], Rel.shape[0]
    Et, Rt = torch.from_numpy(E).cuda(), torch.from_numpy(Rel).cuda()
    flush = torch.empty(512 * 1024 * 1024 // 4, device="cuda")
    for spec in sys.argv[4:]:
        opts = parse(spec)
        with kgc.Join(**opts) as j:
            for _ in range(2):
                j.run(Et, Rt, norm, th)
            st = []
            for _ in range(steps):
                flush.zero_()
                torch.cuda.synchronize()
                j.run(Et, Rt, norm, th)
                st.append(j.stats())
        m = {k: round(statistics.mean(s[k] for s in st), 3) for k in st[0] if k.startswith("ms_")}
        s = st[-1]
        pairs = s["tile_pairs_mine"] * s["query_tile_rows"] * s["tail_tile_rows"]
        print(json.dumps({"opts": spec, "engine": s["engine"], **m, "results": s["results"],
                          "candidates": s["candidates"], "tile_pair_frac": pairs / (N * N * R),
                          "gathered_pair_frac": s["gathered_pairs"] / (N * N * R),
                          "tflops_tiles": 2 * E.shape[1] * (s["gathered_pairs"] or pairs) / (m["ms_tiles"] / 1e3) / 1e12
                          }), flush=True)


if __name__ == "__main__":
    main()
