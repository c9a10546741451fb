"""Time kgc_topk (device inputs, CUDA events on the context's stream) on bench configs.
usage (under gpurun): python scripts/bench_topk.py c2:2:100 c3:2:100 ..."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2307_12059_b200 import kgc  # noqa: E402
from synth import generate_config  # noqa: E402

for spec in sys.argv[1:] or ["c2:2:100"]:
    cfg, norm, k = spec.split(":")
    norm, k = int(norm), int(k)
    E, Rel = generate_config(cfg)
    Et, Rt = torch.from_numpy(E).cuda(), torch.from_numpy(Rel).cuda()
    s = torch.cuda.current_stream()
    with kgc.Join(stream=s.cuda_stream, pivots=8) as j:
        for excl in (False, True):
            j.topk(Et, Rt, norm, k, excl)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(s)
            res = j.topk(Et, Rt, norm, k, excl)
            b.record(s)
            torch.cuda.synchronize()
            st = j.stats()
            print(json.dumps({"config": cfg, "norm": norm, "k": k, "exclude_self": excl,
                              "ms_device": a.elapsed_time(b), "ms_wall": (time.perf_counter() - t0) * 1e3,
                              "join_eps_results": st["results"], "join_ms_total": st["ms_total"],
                              "top1": float(res["dist"][0]), "kth": float(res["dist"][-1])}), flush=True)
