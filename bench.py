"""bench.py -- throughput of the B200 TransE completion join (arXiv 2307.12059).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c2] [--hit 1e-4]

One *step* is one pass of the whole hot path (every SURVEY §8(a) row) over the
synthetic workload: kgc_join with L2 (tcgen05 engine) followed by kgc_join
with L1 (SIMT engine) on the same inputs, each = K1 keys, K2 sorts, K3 tile
ranges + shard split, staging, tile engine, FP64 verify + compaction.

metric = candidate triplets / s = (N * N * R per join, summed over the two
joins) / device time of the step; whole-job value over all ranks (query tiles
are sharded across ranks, tails replicated: strong scaling on a fixed config).

For N > 1 launch with torchrun (one process per GPU, NCCL); the timed region
ends with an NCCL all-reduce of the result counts; times are the max over
ranks.  Inputs are resident in HBM when the timed region starts; L2 is
flushed (512 MiB write) before every timed step, outside the events.
"""
from __future__ import annotations

import argparse
from concurrent.futures import ThreadPoolExecutor
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

from synth import CONFIGS, GENERATOR_VERSION, generate_config, sample_rows  # noqa: E402

METRIC = "candidate triplets/s (N*N*R/time)"
UNIT = "triplets/s"


def load_thresholds():
    return json.loads((ROOT / "configs" / "thresholds.json").read_text())


def load_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        return json.loads(p.read_text()), "measured"
    return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0, "sm_max_mhz": 1965.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self.proc = None
        self.thread = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.thread.join(timeout=2)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}

        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [num(r[1]) for r in self.rows if num(r[1]) is not None]
        mx = [num(r[2]) for r in self.rows if num(r[2]) is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max((num(r[3]) or 0.0) for r in self.rows)}


def ncu_traffic(kernel: str, workload: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, or None."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if not p.exists():
        return None
    try:
        d = json.loads(p.read_text())
        w = d.get(workload, {})
        if kernel in w:
            return w[kernel].get("dram_bytes_per_launch")
        # template arguments beyond the first (tile shapes) may differ between captures: newest matching tag
        base = kernel.rstrip(">").split(",")[0]
        hits = [v for k, v in w.items() if k.split(",")[0].rstrip(">") == base]
        return max(hits, key=lambda v: v.get("tag", ""))["dram_bytes_per_launch"] if hits else None
    except (ValueError, AttributeError, KeyError):
        return None


def element_fraction(join, N, R, K, eps, rows):
    """Element-level Lemma-1 survivors: fraction of (q, t) pairs of the sampled query rows whose
    pivot-distance bound max_k |d(q,p_k) - d(t,p_k)| <= theta (the pairs a per-element filter would
    keep; the tile-granular filter keeps more).  From the keys the join computed (kgc_inspect)."""
    import numpy as np
    kt = join.inspect("tail_keys").reshape(N, K).astype(np.float64)
    kq = join.inspect("query_keys").reshape(R * N, K).astype(np.float64)
    sel = kq[rows]
    keep = 0
    for a in range(0, sel.shape[0], 32):
        diff = np.abs(sel[a:a + 32, None, :] - kt[None, :, :]).max(axis=2)
        keep += int((diff <= eps).sum())
    return keep / (len(rows) * N)


# ------------------------------------------------------------------ reference arm
def run_reference(args, cfg, thresholds):
    """The oracle (plain FP64 CPU brute force) on a bounded sample per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import oracle
    E, Rel = generate_config(args.config)
    N, R, d = cfg.N, cfg.R, cfg.d
    eps = {n: thresholds[args.config][f"L{n}@{args.hit:g}"]["theta"] for n in args.norms}
    rows_per_step = args.ref_rows

    def step(seed):
        rows = sample_rows(N, R, rows_per_step, seed=seed)
        t0 = time.perf_counter()
        for n in args.norms:
            oracle.join(E, Rel, n, eps[n], rows=rows)
        return time.perf_counter() - t0

    for w in range(args.warmup):
        step(1000 + w)
    times = [step(2000 + k) for k in range(args.steps)]
    trip = rows_per_step * N * len(args.norms)
    value = trip * len(times) / sum(times)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_name(args, cfg), "sample": f"{rows_per_step} seeded (h,r) rows x all {N} "
                   f"tails per step, norms {args.norms}"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.threads_used(), "kind": "oracle",
                         "sample": f"{rows_per_step} (h,r) rows x {N} tails x norms {args.norms} per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_name(args, cfg):
    return (f"{cfg.name} ({cfg.note}): N={cfg.N} R={cfg.R} d={cfg.d}, TransE norms {args.norms}, "
            f"theta at hit rate {args.hit:g}, {cfg.dist} embeddings ({GENERATOR_VERSION}, seed {cfg.seed})")


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg, thresholds):
    import torch
    import torch.distributed as dist

    from paper_2307_12059_b200 import kgc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"warning: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()

    N, R, d = cfg.N, cfg.R, cfg.d
    eps = {n: float(thresholds[args.config][f"L{n}@{args.hit:g}"]["theta"]) for n in args.norms}
    # inputs: rank 0 generates, NCCL broadcast to the other ranks (outside the timed region)
    if rank == 0:
        E_h, Rel_h = generate_config(args.config)
        Et = torch.from_numpy(E_h).to(dev)
        Rt = torch.from_numpy(Rel_h).to(dev)
    else:
        E_h = Rel_h = None
        Et = torch.empty((N, d), dtype=torch.float32, device=dev)
        Rt = torch.empty((R, d), dtype=torch.float32, device=dev)
    if world > 1:
        dist.broadcast(Et, 0)
        dist.broadcast(Rt, 0)
    if E_h is None:
        E_h, Rel_h = Et.cpu().numpy(), Rt.cpu().numpy()
    torch.cuda.synchronize()

    # the joins of one step (one per norm) run concurrently: one context, stream and host thread
    # each (a context is single-threaded; kgc_join blocks its thread at its two host syncs, so
    # the other join fills those gaps); --sequential runs them one after the other on one stream
    conc = len(args.norms) > 1 and not args.sequential
    jstream = {n: (torch.cuda.Stream(dev) if conc else stream) for n in args.norms}
    pool = ThreadPoolExecutor(len(args.norms)) if conc else None

    def run_joins(fn):
        """fn(n) for every norm, concurrently on the norms' streams, ordered after / before `stream`."""
        if not conc:
            return [fn(n) for n in args.norms]
        ev0 = torch.cuda.Event()
        ev0.record(stream)
        for n in args.norms:
            jstream[n].wait_event(ev0)
        out = [f.result() for f in [pool.submit(fn, n) for n in args.norms]]
        for n in args.norms:
            ev = torch.cuda.Event()
            ev.record(jstream[n])
            stream.wait_event(ev)
        return out

    joins = {n: kgc.Join(device=local, rank=rank, world=world, pivots=args.pivots, split=args.split, tail_shard=args.tail_shard, stream=jstream[n].cuda_stream)
             for n in args.norms}
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    counts = torch.zeros(len(args.norms), dtype=torch.int64, device=dev)

    def step():
        cs = run_joins(lambda n: joins[n].run(Et, Rt, n, eps[n]))
        for i, c in enumerate(cs):
            counts[i] = c
        if world > 1:
            dist.all_reduce(counts)

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()

    # ---- timed region (device time, CUDA events on the launching stream)
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    phase = {n: {} for n in args.norms}
    launches = 0
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        for k in range(args.steps):
            flush.zero_()                      # L2 flush (> 126 MB), outside the events
            starts[k].record(stream)
            step()
            ends[k].record(stream)
            for n in args.norms:
                st = joins[n].stats()
                launches += st["launches"]
                for key in ("ms_total", "ms_h2d", "ms_keys", "ms_sort", "ms_ranges", "ms_stage", "ms_tiles",
                            "ms_recheck"):
                    phase[n].setdefault(key, []).append(st[key])
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    wall = time.perf_counter() - wall0
    ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    trip_per_step = float(N) * N * R * len(args.norms)
    value = trip_per_step / (ms_per_step / 1e3)
    results_total = int(counts.sum().item())
    stats_last = {n: joins[n].stats() for n in args.norms}

    # ---- roofline of the dominant kernel (per-phase CUDA events inside libkgc)
    peaks, peak_src = load_peaks()
    kernels = []
    for n in args.norms:
        st = stats_last[n]
        t_tiles = statistics.mean(phase[n]["ms_tiles"]) / 1e3
        pairs = st["tile_pairs_mine"] * st["query_tile_rows"] * st["tail_tile_rows"]
        if st["engine"] == 5:   # gathered tails: the pairs left after the per-tail pivot test (padding excluded)
            pairs = st["gathered_pairs"]
        flops = 2.0 * d * pairs
        if n == 2:
            tc = st["tail_tile_rows"] == 256
            peak = peaks["bf16_tflops"] * (1.1 / 2.25) if tc else \
                148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12 * 2
            kname = ("tiles_tc2_kernel (L2, tcgen05.mma.cta_group::2 kind::tf32)" if st["engine"] == 4 else
                     "tiles_tc_kernel (L2, tcgen05 kind::tf32)") if tc else "tiles_simt_kernel<2>"
            kernels.append({"kernel": kname,
                            "bound": "tensor" if tc else "alu", "ms": t_tiles * 1e3,
                            "achieved": flops / t_tiles / 1e12, "peak": peak, "unit": "TFLOP/s",
                            "peak_note": (f"{peak_src} bf16 burst {peaks['bf16_tflops']} x nominal tf32/bf16 "
                                          "1.1/2.25") if tc else "148 SM x 128 FP32 lanes x FFMA(2 flop) x clock"})
        else:
            peak = 148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
            kname = "tiles_gather_kernel<1> (L1, gathered tails)" if st["engine"] == 5 else "tiles_simt_kernel<1> (L1)"
            kernels.append({"kernel": kname, "bound": "alu", "ms": t_tiles * 1e3,
                            "achieved": flops / t_tiles / 1e12, "peak": peak, "unit": "TFLOP/s",
                            "peak_note": "148 SM x 128 FP32 lanes x 1 FADD/clk x sm_max_mhz (|q-t| = 2 FADD = 2 flop)"})
        if n == 1:
            # the L1 path's HBM use (BASELINE north_star asks for it): ncu dram bytes of the tile kernel /
            # its event time; operand bytes the bulk copies move (L2 -> SM) per the same time
            k1 = kernels[-1]
            dram = ncu_traffic(k1["kernel"].split()[0], args.config)
            # operand bytes per computed pair: (query rows + tail rows) x Kpad x 4 per 64 x 64 block
            opb = pairs * (st["query_tile_rows"] + st["tail_tile_rows"]) * ((d + 7) // 8 * 8) * 4 / \
                (st["query_tile_rows"] * st["tail_tile_rows"])
            k1["hbm_gbs"] = dram / t_tiles / 1e9 if dram else None
            k1["hbm_frac"] = (dram / t_tiles / 1e9) / peaks["hbm_gbs"] if dram else None
            k1["operand_gbs_l2_to_sm"] = opb / t_tiles / 1e9
        for key, name in (("ms_keys", "K1 keys"), ("ms_sort", "K2 sort"), ("ms_ranges", "K3 ranges"),
                          ("ms_stage", "stage"), ("ms_recheck", "K6 verify")):
            ent = {"kernel": f"{name} (L{n})", "ms": statistics.mean(phase[n][key])}
            if key == "ms_keys":
                # algorithmic HBM bytes of the precompute: read E and Rel, write N*R + N keys x K pivots
                Kp = st["pivots_used"]
                byts = (N * d + R * d) * 4 + (N * R + N) * Kp * 4
                ent.update({"bound": "hbm", "achieved_gbs": byts / (ent["ms"] / 1e3) / 1e9,
                            "peak_gbs": peaks["hbm_gbs"],
                            "frac": byts / (ent["ms"] / 1e3) / 1e9 / peaks["hbm_gbs"],
                            "note": "phase time incl. pivot choice and both key kernels; E is L2-resident"})
            kernels.append(ent)
    dom = max((k for k in kernels if "achieved" in k), key=lambda k: k["ms"])
    wl = workload_name(args, cfg)
    traffic = ncu_traffic(dom["kernel"].split()[0], args.config)
    roofline = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
                "frac": dom["achieved"] / dom["peak"], "traffic": traffic, "kernel": dom["kernel"],
                "peak_source": dom["peak_note"]}

    # ---- end to end through the public C ABI with HOST buffers
    e2e = None
    if not args.no_e2e:
        E_pin = torch.from_numpy(E_h).pin_memory()
        R_pin = torch.from_numpy(Rel_h).pin_memory()
        out_pin = {n: torch.empty((max(1, stats_last[n]["results"]) * 2, 4), dtype=torch.int32).pin_memory()
                   for n in args.norms}
        e2e_joins = {n: kgc.Join(device=local, rank=rank, world=world, pivots=args.pivots, split=args.split, tail_shard=args.tail_shard,
                                 stream=jstream[n].cuda_stream) for n in args.norms}
        h2d = d2h = 0

        def e2e_one(n):
            j = e2e_joins[n]
            kgc.kgc_join(j.ctx, E_pin, R_pin, N, R, d, n, eps[n])
            cnt = kgc.kgc_results(j.ctx)
            if cnt > out_pin[n].shape[0]:
                out_pin[n] = torch.empty((cnt * 2, 4), dtype=torch.int32).pin_memory()
            kgc.kgc_results(j.ctx, out_pin[n], cnt)
            return cnt

        def e2e_step():
            nonlocal h2d, d2h
            for cnt in run_joins(e2e_one):
                h2d += E_pin.numel() * 4 + R_pin.numel() * 4
                d2h += cnt * 16
        e2e_step()
        torch.cuda.synchronize()
        h2d = d2h = 0
        if world > 1:
            dist.barrier()
        s0 = torch.cuda.Event(enable_timing=True)
        s1 = torch.cuda.Event(enable_timing=True)
        s0.record(stream)
        for _ in range(args.steps):
            e2e_step()
        s1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([s0.elapsed_time(s1)], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        e2e_ms = float(te.item()) / args.steps
        e2e = {"value": trip_per_step / (e2e_ms / 1e3), "unit": UNIT, "ms_per_step": e2e_ms,
               "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
               "path": "kgc_join(host pinned E, Rel) + kgc_results(host pinned) per norm"}
        for j in e2e_joins.values():
            j.close()

    # ---- CPU baseline: the oracle on a bounded sample, rank 0 at N=1 only
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from oracle import oracle
        probe_rows = sample_rows(N, R, 32, seed=99)
        t0 = time.perf_counter()
        for n in args.norms:
            oracle.join(E_h, Rel_h, n, eps[n], rows=probe_rows)
        per_row = (time.perf_counter() - t0) / 32
        S = int(min(max(64, args.cpu_seconds / max(per_row, 1e-9)), N * R))
        rows = sample_rows(N, R, S, seed=100)
        t0 = time.perf_counter()
        for n in args.norms:
            oracle.join(E_h, Rel_h, n, eps[n], rows=rows)
        tcpu = time.perf_counter() - t0
        cpu = {"value": S * N * len(args.norms) / tcpu, "unit": UNIT, "cores": oracle.threads_used(),
               "kind": "oracle", "seconds": tcpu,
               "sample": f"{S} seeded (h,r) rows x all {N} tails, norms {args.norms} (FP64 brute force, C + OpenMP)"}

    elem = None
    if rank == 0 and world == 1:
        rows = sample_rows(N, R, 256, seed=5)
        elem = {f"L{n}": element_fraction(joins[n], N, R, stats_last[n]["pivots_used"], eps[n], rows)
                for n in args.norms}
    for j in joins.values():
        j.close()
    clocks = clk.summary()
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32",
            "dtype_detail": "L2 filter tcgen05 kind::tf32 (FP32 accumulate) + rigorous guard band; L1 filter FP32 "
                            "SIMT on gathered tails; every emitted triplet re-checked in FP64",
            "data": "synthetic",
            "config": {"workload": wl, "N": N, "R": R, "d": d, "norms": args.norms, "eps": eps, "hit_rate": args.hit,
                       "parallelism": (f"tail partitions x{world}, every query on every rank" if args.tail_shard else
                                       f"query-tile shards x{world} ({['rank-local', 'cost-balanced', 'cyclic'][args.split]} "
                                       f"split), tails replicated"),
                       "joins": ("concurrent: one context, stream and host thread per norm" if conc else
                                 "sequential on one stream"),
                       "pivots": args.pivots,
                       "l2_cache": "flushed (512 MiB write) before every timed step, outside the timed events"},
            "result_triplets_per_step": results_total,
            "result_triplets_per_s": results_total / (ms_per_step / 1e3),
            "pruned_tile_fraction": {f"L{n}": 1 - stats_last[n]["tile_pairs_surviving"] /
                                     max(1, stats_last[n]["tile_pairs_total"]) for n in args.norms},
            "candidates_per_result": {f"L{n}": stats_last[n]["candidates"] / max(1, stats_last[n]["results"])
                                      for n in args.norms},
            "surviving_pair_fraction_tiles": {f"L{n}": stats_last[n]["tile_pairs_surviving"] *
                                              stats_last[n]["query_tile_rows"] * stats_last[n]["tail_tile_rows"] /
                                              max(1.0, float(N) * N * R) for n in args.norms},
            "surviving_pair_fraction_gathered": {f"L{n}": stats_last[n]["gathered_pairs"] / max(1.0, float(N) * N * R)
                                                 for n in args.norms if stats_last[n]["engine"] == 5},
            "surviving_pair_fraction_elements_sampled": elem,
            "roofline": roofline, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": launches, "clocks": clocks, "wall_s_timed_region": wall,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def run_emulated_ranks(args, cfg, thresholds):
    """Every shard of a W-rank run, one after the other on one GPU (device time per
    shard, CUDA events, L2 flushed before each).  The data path has no collective,
    so max over shards projects the N=W step time (NCCL count all-reduce excluded)."""
    import torch

    from paper_2307_12059_b200 import kgc
    W = args.emulate_ranks
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    N, R, d = cfg.N, cfg.R, cfg.d
    eps = {n: float(thresholds[args.config][f"L{n}@{args.hit:g}"]["theta"]) for n in args.norms}
    E_h, Rel_h = generate_config(args.config)
    Et, Rt = torch.from_numpy(E_h).to(dev), torch.from_numpy(Rel_h).to(dev)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    out = {"emulated_ranks": W, "config": args.config, "pivots": args.pivots, "shard_ms": []}
    for rank in range(W):
        joins = {n: kgc.Join(device=0, rank=rank, world=W, pivots=args.pivots, split=args.split, tail_shard=args.tail_shard, stream=stream.cuda_stream)
                 for n in args.norms}
        for _ in range(max(1, args.warmup)):
            for n in args.norms:
                joins[n].run(Et, Rt, n, eps[n])
        times = []
        for _ in range(args.steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for n in args.norms:
                joins[n].run(Et, Rt, n, eps[n])
            b.record(stream)
            torch.cuda.synchronize()
            times.append(a.elapsed_time(b))
        out["shard_ms"].append(statistics.mean(times))
        ph = {f"L{n}": {k: round(v, 3) for k, v in joins[n].stats().items()
                        if k.startswith("ms_") or k in ("launches", "work_items_mine", "tile_pairs_mine",
                                                         "gathered_pairs", "candidates")}
              for n in args.norms}
        if rank == 0:
            out["rank0_phases"] = ph
        out.setdefault("phases", []).append(ph)
        for j in joins.values():
            j.close()
    ms = max(out["shard_ms"])
    out["projected_ms_per_step"] = ms
    out["projected_value"] = float(N) * N * R * len(args.norms) / (ms / 1e3)
    print(json.dumps(out), flush=True)
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--hit", type=float, default=1e-4)
    ap.add_argument("--norms", default="2,1", help="norms joined per step, e.g. '2,1' or '2'")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sequential", action="store_true", help="run the step's joins one after the other")
    ap.add_argument("--tail-shard", type=int, default=0,
                    help="world > 1: 1 = partition-based join (rank k holds tails [kN/W, (k+1)N/W), every query)")
    ap.add_argument("--split", default="auto",
                    help="world > 1: 0 = rank-local split, 1 = global cost-balanced, 2 = cyclic; auto = best "
                         "measured per config (c2: 2, its hits concentrate in a few relations)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-rows", type=int, default=256, help="(h,r) rows per reference step")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="diagnostic: on ONE GPU run each of W shards in turn and print the per-shard device times "
                         "(projects the N=W device time; not the official line)")
    ap.add_argument("--pivots", default="auto",
                    help="1 = the paper's single pivot; 2..8 = multi-pivot pruning; auto = best measured per config")
    args = ap.parse_args()
    args.norms = [int(x) for x in args.norms.split(",")]
    # Best measured pivot count per workload: multi-pivot pruning pays on c2 / c4,
    # the paper's single pivot is faster on c3 (its extra keys/sort cost exceeds the pruning gain).
    best_pivots = {"c1": 1, "c2": 8, "c3": 1, "c4": 8, "c5": 8}
    args.pivots = best_pivots.get(args.config, 1) if args.pivots == "auto" else int(args.pivots)
    args.split = {"c2": 2}.get(args.config, 0) if args.split == "auto" else int(args.split)
    cfg = CONFIGS[args.config]
    thresholds = load_thresholds()
    if args.impl == "reference":
        return run_reference(args, cfg, thresholds)
    if args.emulate_ranks:
        return run_emulated_ranks(args, cfg, thresholds)
    return run_ours(args, cfg, thresholds)


if __name__ == "__main__":
    sys.exit(main())
