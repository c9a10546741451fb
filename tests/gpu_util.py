"""Helpers for the GPU parity tests: run libkgc through its C ABI, compare with
the oracle on the same seeded inputs."""
from __future__ import annotations

import numpy as np

from oracle import oracle as orc


def gpu_join(E, Rel, norm, eps, device_inputs=True, **opts):
    import torch

    from paper_2307_12059_b200 import kgc
    with kgc.Join(**opts) as j:
        if device_inputs:
            Et = torch.from_numpy(np.ascontiguousarray(E)).cuda()
            Rt = torch.from_numpy(np.ascontiguousarray(Rel)).cuda()
            torch.cuda.synchronize()
            j.run(Et, Rt, norm, eps)
        else:
            j.run(np.ascontiguousarray(E), np.ascontiguousarray(Rel), norm, eps)
        return j.results(), j.stats()


def restrict_rows(res, rows, R):
    key = res["h"].astype(np.int64) * R + res["r"]
    return res[np.isin(key, rows)]


def check_parity(E, Rel, norm, eps, gpu_res, rows=None, band=1e-4, dist_rel=1e-5):
    """tight <= gpu <= loose, no duplicates, distances within dist_rel."""
    R = Rel.shape[0]
    loose = orc.join(E, Rel, norm, float(eps) * (1 + band), rows=rows)
    g = gpu_res if rows is None else restrict_rows(gpu_res, rows, R)
    rep = orc.compare(g, loose, float(eps), band_rel=band, dist_rel=dist_rel)
    assert rep["duplicates"] == 0, rep
    assert rep["missing"] == 0, rep
    assert rep["extra"] == 0, rep
    assert rep["max_dist_rel_err"] <= dist_rel, rep
    return rep


def theta_for(E, Rel, norm, hit_rate, rows=None):
    if rows is None:
        rows = np.arange(E.shape[0] * Rel.shape[0])
    try:
        th, _ = orc.calibrate_theta(E, Rel, norm, hit_rate, rows)
        return th
    except RuntimeError:
        # tiny instances: middle of the widest gap near the requested quantile
        D = np.sort(orc.dist_rows(E, Rel, norm, rows).ravel())
        k = max(1, int(round(hit_rate * D.size)))
        if D.size == 1:
            return float(np.float32(D[0] * 1.5 + 0.1))
        lo = max(0, k - 3)
        hi = min(D.size - 1, k + 3)
        g = max(range(lo, hi), key=lambda a: D[a + 1] - D[a])
        return float(np.float32(0.5 * (D[g] + D[g + 1])))


def keyset(a):
    return set(zip(a["h"].tolist(), a["r"].tolist(), a["t"].tolist()))
