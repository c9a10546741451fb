"""bench.py -- throughput of the B200 TransE completion join (arXiv 2307.12059).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config c4] [--hit 1e-5]

One *step* is one pass of the whole hot path (every SURVEY §8(a) row) over the
synthetic workload: kgc_join per norm of the workload on the same inputs, each =
(N > 1: E/Rel broadcast from rank 0) K1 keys, K2 sorts, K3 tile ranges + shard
split, staging, tile engine, FP64 verify + compaction (and the count all-reduce).

Default workload: c4 (YAGO3-10-shaped, N=123182, R=37, d=200, TransE L2, theta at
hit rate 1e-5), the largest BASELINE.json config that fits one GPU's
single-GPU line (c5 is the 8-GPU config).  The same JSON line also carries
`extra_workloads`: the c2 L2+L1 step (WN18-shaped, both norms) and the c3
theta sweep (FB15k-shaped, hit rates 1e-6..1e-3; the analogue of the paper's
epsilon sweep), each timed the same way, and
`projected_scaling`: every shard of a 2/4/8-rank c4 and c5 join (split 3) in turn
on this GPU, max shard device time -- a projection, not a multi-GPU measurement.

metric = candidate triplets / s = (N * N * R per join, summed over the joins)
/ device time of the step; whole-job value over all ranks (query tiles are
sharded across ranks, tails replicated: strong scaling on a fixed config).

--gpus N > 1 without a launcher re-executes itself under torch.distributed.run
(one process per GPU, NCCL, 127.0.0.1); under torchrun WORLD_SIZE must equal
--gpus.  Times are the max over ranks.  Inputs are resident in HBM (on rank 0)
when the timed region starts; L2 is flushed (512 MiB write) before every timed
step, outside the events.
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
        # template arguments (tile shapes) differ between captures: the newest capture of the same kernel
        base = kernel.split("<")[0]
        hits = [v for k, v in w.items() if k.split("<")[0] == base]
        return hits[-1]["dram_bytes_per_launch"] if hits else None  # the last capture written
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
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": oracle.threads_used(), "cpu_model": cpu_model(),
                         "kind": "oracle",
                         "sample": f"{rows_per_step} (h,r) rows x {N} tails x norms {args.norms} per step"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def workload_name(args, cfg):
    return (f"{cfg.name} ({cfg.note}): N={cfg.N} R={cfg.R} d={cfg.d}, TransE norms {args.norms}, "
            f"theta at hit rate {args.hit:g}, {cfg.dist} embeddings ({GENERATOR_VERSION}, seed {cfg.seed})")


# Best measured settings per workload: with the FP64-factorised L2 keys (query keys
# never materialised) many pivots cut the surviving tile pairs (c4: 4.76% at 8, 1.01% at 64, 0.37% at
# 96); whole join c4 17.4 (8) -> 8.1 (64) -> 6.9 ms (96), c5 1460 -> 524 -> 443 ms (128), c3 10.4 (one
# pivot) -> 7.0 ms (64); c2 takes 32 (the L1 keys support at most 32); the cyclic split spreads c2's
# hit-dense relations.
BEST_PIVOTS = {"c1": 1, "c2": 32, "c3": 64, "c4": 96, "c5": 128}
BEST_SPLIT = {"c2": 2, "c3": 3, "c4": 3, "c5": 3}
DEFAULT_HIT = {"c1": 1e-3, "c2": 1e-4, "c3": 1e-5, "c4": 1e-5, "c5": 1e-6}
DEFAULT_NORMS = {"c1": "2,1", "c2": "2,1", "c3": "2", "c4": "2", "c5": "2"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


class StepRunner:
    """The joins of one step: one libkgc context per norm.  With two norms they run
    concurrently, each on its own stream and host thread (a context is single-threaded
    and kgc_join blocks its thread at two host syncs, so the other join fills those gaps);
    `sequential` runs them one after the other on `stream`."""

    def __init__(self, torch, kgc, dev, stream, norms, eps, rank, world, pivots, split, tail_shard, sequential):
        self.torch, self.stream, self.norms, self.eps = torch, stream, norms, eps
        self.conc = len(norms) > 1 and not sequential
        self.jstream = {n: (torch.cuda.Stream(dev) if self.conc else stream) for n in norms}
        self.pool = ThreadPoolExecutor(len(norms)) if self.conc else None
        self.opts = dict(device=dev.index, rank=rank, world=world, pivots=pivots, split=split, tail_shard=tail_shard)
        self.kgc = kgc
        self.joins = {n: kgc.Join(stream=self.jstream[n].cuda_stream, **self.opts) for n in norms}

    def new_joins(self):
        return {n: self.kgc.Join(stream=self.jstream[n].cuda_stream, **self.opts) for n in self.norms}

    def run_joins(self, fn):
        """fn(n) for every norm, concurrently on the norms' streams, ordered after / before `stream`."""
        torch = self.torch
        if not self.conc:
            return [fn(n) for n in self.norms]
        ev0 = torch.cuda.Event()
        ev0.record(self.stream)
        for n in self.norms:
            self.jstream[n].wait_event(ev0)
        out = [f.result() for f in [self.pool.submit(fn, n) for n in self.norms]]
        for n in self.norms:
            ev = torch.cuda.Event()
            ev.record(self.jstream[n])
            self.stream.wait_event(ev)
        return out

    def close(self):
        for j in self.joins.values():
            j.close()
        if self.pool:
            self.pool.shutdown()


PHASES = ("ms_total", "ms_h2d", "ms_keys", "ms_sort", "ms_ranges", "ms_stage", "ms_tiles", "ms_recheck")


def timed_steps(torch, stream, step, steps, flush, barrier=None):
    """`steps` timed steps (CUDA events on `stream`, L2 flushed before each outside the events);
    returns (total ms, per-step per-norm stats list)."""
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    stats = []
    if barrier:
        barrier()
    torch.cuda.synchronize()
    for k in range(steps):
        flush.zero_()                      # L2 flush (> 126 MB), outside the events
        starts[k].record(stream)
        stats.append(step())
        ends[k].record(stream)
    torch.cuda.synchronize()
    if barrier:
        barrier()
    return sum(s.elapsed_time(e) for s, e in zip(starts, ends)), stats


def kernel_table(stats_steps, norms, d, peaks, peak_src, config, N, R):
    """Per-kernel device times (libkgc's per-phase CUDA events on the launching stream) and the
    roofline of each tile kernel: algorithmic work per unit x units per launch / mean duration."""
    last = stats_steps[-1]
    kernels = []
    for n in norms:
        st = last[n]
        mean = {k: statistics.mean(s[n][k] for s in stats_steps) for k in PHASES}
        t_tiles = mean["ms_tiles"] / 1e3
        pairs = st["tile_pairs_mine"] * st["query_tile_rows"] * st["tail_tile_rows"]
        if st["engine"] == 5:   # gathered tails: the pairs left after the per-tail pivot test (padding excluded)
            pairs = st["gathered_pairs"]
        flops = 2.0 * d * pairs
        alu = 148 * 128 * peaks.get("sm_max_mhz", 1965.0) * 1e6 / 1e12
        if n == 2:
            tc = st["engine"] in (1, 4, 6, 7, 8)  # tensor-core engines (kgc.h kgc_stats_t.engine)
            peak = peaks["bf16_tflops"] * (1.1 / 2.25) if tc else 2 * alu
            kname = ("tiles_tc2_kernel (L2, tcgen05.mma.cta_group::2 kind::tf32)" if st["engine"] in (4, 8) else
                     "tiles_tc_kernel (L2, tcgen05 kind::tf32)") if tc else "tiles_simt_kernel<2>"
            ent = {"kernel": kname, "bound": "tensor" if tc else "alu", "ms": t_tiles * 1e3,
                   "achieved": flops / t_tiles / 1e12 if t_tiles > 0 else 0.0, "peak": peak, "unit": "TFLOP/s",
                   "work": f"2*d flops x {pairs:.4g} (query, tail) pairs in surviving {st['query_tile_rows']}x"
                           f"{st['tail_tile_rows']} tiles",
                   "peak_note": (f"{peak_src} bf16 burst {peaks['bf16_tflops']} x nominal tf32/bf16 1.1/2.25")
                   if tc else "148 SM x 128 FP32 lanes x FFMA(2 flop) x clock"}
        else:
            kname = "tiles_gather_kernel<1> (L1, gathered tails)" if st["engine"] == 5 else "tiles_simt_kernel<1> (L1)"
            ent = {"kernel": kname, "bound": "alu", "ms": t_tiles * 1e3,
                   "achieved": flops / t_tiles / 1e12 if t_tiles > 0 else 0.0, "peak": alu, "unit": "TFLOP/s",
                   "work": f"2*d FP32 ops x {pairs:.4g} computed (query, tail) pairs",
                   "peak_note": "148 SM x 128 FP32 lanes x 1 FADD/clk x sm_max_mhz (|q-t| = 2 FADD = 2 flop)"}
            # the L1 path's HBM use (BASELINE north_star asks for it): ncu dram bytes of the tile kernel /
            # its event time; operand bytes the copies move (L2 -> SM) per the same time
            dram = ncu_traffic(kname.split()[0], config)
            opb = pairs * (st["query_tile_rows"] + st["tail_tile_rows"]) * ((d + 7) // 8 * 8) * 4 / \
                (st["query_tile_rows"] * st["tail_tile_rows"])
            ent["hbm_gbs"] = dram / t_tiles / 1e9 if dram and t_tiles > 0 else None
            ent["hbm_frac"] = ent["hbm_gbs"] / peaks["hbm_gbs"] if ent["hbm_gbs"] else None
            ent["operand_gbs_l2_to_sm"] = opb / t_tiles / 1e9 if t_tiles > 0 else None
        ent["frac"] = ent["achieved"] / ent["peak"]
        kernels.append(ent)
        for key, name in (("ms_keys", "K1 keys"), ("ms_sort", "K2 sort"), ("ms_ranges", "K3 ranges"),
                          ("ms_stage", "stage"), ("ms_recheck", "K6 verify")):
            e = {"kernel": f"{name} (L{n})", "ms": mean[key]}
            if key == "ms_keys" and mean[key] > 0:
                # algorithmic HBM bytes of the precompute: read E and Rel, write N*R + N keys x K pivots
                Kp = st["pivots_used"]
                byts = (N * d + R * d) * 4 + (N * R + N) * Kp * 4
                e.update({"bound": "hbm", "achieved_gbs": byts / (mean[key] / 1e3) / 1e9, "peak_gbs": peaks["hbm_gbs"],
                          "frac": byts / (mean[key] / 1e3) / 1e9 / peaks["hbm_gbs"],
                          "note": "phase time incl. pivot choice and both key kernels; E is L2-resident"})
            if key == "ms_recheck":
                e["candidates"] = st["candidates"]
            kernels.append(e)
    return kernels


def measure_workload(torch, kgc, dev, stream, name, norms, hit, steps, warmup, thresholds, flush, sequential=False):
    """One extra workload on this GPU (world 1), timed like the headline: {value, ms_per_step, ...}."""
    cfg = CONFIGS[name]
    E_h, Rel_h = generate_config(name)
    Et, Rt = torch.from_numpy(E_h).to(dev), torch.from_numpy(Rel_h).to(dev)
    eps = {n: float(thresholds[name][f"L{n}@{hit:g}"]["theta"]) for n in norms}
    runner = StepRunner(torch, kgc, dev, stream, norms, eps, 0, 1, BEST_PIVOTS.get(name, 1), 0, 0, sequential)

    def step():
        runner.run_joins(lambda n: runner.joins[n].run(Et, Rt, n, eps[n]))
        return {n: runner.joins[n].stats() for n in norms}

    for _ in range(warmup):
        step()
    ms, stats = timed_steps(torch, stream, step, steps, flush)
    runner.close()
    ms_step = ms / steps
    trip = float(cfg.N) * cfg.N * cfg.R * len(norms)
    peaks, peak_src = load_peaks()
    kern = kernel_table(stats, norms, cfg.d, peaks, peak_src, name, cfg.N, cfg.R)
    tiles = [k for k in kern if "achieved" in k]
    dom = max(tiles, key=lambda k: k["ms"])
    res = sum(stats[-1][n]["results"] for n in norms)
    return {"workload": f"{name}: N={cfg.N} R={cfg.R} d={cfg.d}, norms {norms}, hit rate {hit:g}",
            "value": trip / (ms_step / 1e3), "unit": UNIT, "ms_per_step": ms_step, "steps": steps,
            "eps": eps, "result_triplets_per_step": res,
            "pruned_tile_fraction": {f"L{n}": 1 - stats[-1][n]["tile_pairs_surviving"] /
                                     max(1, stats[-1][n]["tile_pairs_total"]) for n in norms},
            "dominant_kernel": {"kernel": dom["kernel"], "ms": dom["ms"], "frac": dom["frac"], "bound": dom["bound"]},
            "phases_ms": {k["kernel"]: round(k["ms"], 4) for k in kern}}


# ------------------------------------------------------------------ our arm
def run_ours(args, cfg, thresholds):
    import torch
    import torch.distributed as dist

    from paper_2307_12059_b200 import kgc

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE {world}", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream()
    barrier = (lambda: dist.barrier()) if world > 1 else None

    N, R, d = cfg.N, cfg.R, cfg.d
    eps = {n: float(thresholds[args.config][f"L{n}@{args.hit:g}"]["theta"]) for n in args.norms}
    # inputs: resident on rank 0; every step starts with their NCCL broadcast to the other ranks
    # (inside the timed region)
    if rank == 0:
        E_h, Rel_h = generate_config(args.config)
        Et = torch.from_numpy(E_h).to(dev)
        Rt = torch.from_numpy(Rel_h).to(dev)
    else:
        E_h = Rel_h = None
        Et = torch.empty((N, d), dtype=torch.float32, device=dev)
        Rt = torch.empty((R, d), dtype=torch.float32, device=dev)
    torch.cuda.synchronize()

    runner = StepRunner(torch, kgc, dev, stream, args.norms, eps, rank, world, args.pivots, args.split,
                        args.tail_shard, args.sequential)
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    counts = torch.zeros(len(args.norms), dtype=torch.int64, device=dev)

    def step():
        if world > 1:
            dist.broadcast(Et, 0)
            dist.broadcast(Rt, 0)
        cs = runner.run_joins(lambda n: runner.joins[n].run(Et, Rt, n, eps[n]))
        for i, c in enumerate(cs):
            counts[i] = c
        if world > 1:
            dist.all_reduce(counts)
        return {n: runner.joins[n].stats() for n in args.norms}

    for _ in range(max(args.warmup, 0)):
        step()
    torch.cuda.synchronize()
    if E_h is None:
        E_h, Rel_h = Et.cpu().numpy(), Rt.cpu().numpy()

    # ---- timed region (device time, CUDA events on the launching stream, max over ranks)
    wall0 = time.perf_counter()
    with ClockSampler(local) as clk:
        ms, stats_steps = timed_steps(torch, stream, step, args.steps, flush, barrier)
    wall = time.perf_counter() - wall0
    launches = sum(s[n]["launches"] for s in stats_steps for n in args.norms)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_per_step = ms_max / args.steps
    trip_per_step = float(N) * N * R * len(args.norms)
    value = trip_per_step / (ms_per_step / 1e3)
    results_total = int(counts.sum().item())
    stats_last = stats_steps[-1]

    peaks, peak_src = load_peaks()
    kernels = kernel_table(stats_steps, args.norms, d, peaks, peak_src, args.config, N, R)
    dom = max((k for k in kernels if "achieved" in k), key=lambda k: k["ms"])
    wl = workload_name(args, cfg)
    traffic = ncu_traffic(dom["kernel"].split()[0], args.config)
    roofline = {"bound": dom["bound"], "achieved": dom["achieved"], "peak": dom["peak"], "unit": dom["unit"],
                "frac": dom["achieved"] / dom["peak"], "traffic": traffic, "kernel": dom["kernel"],
                "work": dom["work"], "peak_source": dom["peak_note"],
                "traffic_note": "dram__bytes_read.sum + dram__bytes_write.sum per launch from the committed ncu "
                                "--set full capture (profiles/ncu_traffic.json)"}

    # ---- end to end through the public C ABI with HOST buffers
    e2e = None
    if not args.no_e2e:
        E_pin = torch.from_numpy(E_h).pin_memory()
        R_pin = torch.from_numpy(Rel_h).pin_memory()
        out_pin = {n: torch.empty((max(1, stats_last[n]["results"]) * 2, 4), dtype=torch.int32).pin_memory()
                   for n in args.norms}
        e2e_joins = runner.new_joins()
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
            for cnt in runner.run_joins(e2e_one):
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
               "path": "kgc_join(host pinned E, Rel) + kgc_results(host pinned) per norm, every rank"}
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
               "cpu_model": cpu_model(), "kind": "oracle", "seconds": tcpu,
               "sample": f"{S} seeded (h,r) rows x all {N} tails, norms {args.norms} (FP64 brute force, C + OpenMP)"}

    elem = None
    if rank == 0 and world == 1 and not args.no_extras:
        rows = sample_rows(N, R, 128 if N > 50000 else 256, seed=5)
        elem = {f"L{n}": element_fraction(runner.joins[n], N, R, stats_last[n]["pivots_used"], eps[n], rows)
                for n in args.norms}
    runner.close()

    # ---- extra workloads (same GPU, same timing rules): c2 both norms, c3 theta sweep
    extras = None
    if rank == 0 and world == 1 and not args.no_extras:
        extras = []
        plan = [("c2", [2, 1], 1e-4)] + [("c3", [2], h) for h in (1e-6, 1e-5, 1e-4, 1e-3)]
        for name, norms, hit in plan:
            if name == args.config and norms == args.norms and hit == args.hit:
                continue
            extras.append(measure_workload(torch, kgc, dev, stream, name, norms, hit, args.extra_steps, 3,
                                           thresholds, flush))
    scaling = None
    if rank == 0 and world == 1 and not args.no_extras and not args.no_scaling:
        scaling = projected_scaling(torch, kgc, dev, stream, thresholds, flush)
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
                                       f"query-tile shards x{world} ({['rank-local', 'cost-balanced', 'cyclic', 'spatial block-cyclic heads'][args.split]} "
                                       f"split), tails replicated; E/Rel NCCL-broadcast from rank 0 every step"),
                       "joins": ("concurrent: one context, stream and host thread per norm" if runner.conc else
                                 "one context per norm on one stream"),
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
            "extra_workloads": extras,
            "projected_scaling": scaling,
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


def projected_scaling(torch, kgc, dev, stream, thresholds, flush, names=("c4", "c5"), Ws=(2, 4, 8), steps=3):
    """Projected multi-GPU device times (diagnostic, one GPU): every shard of a W-rank join in turn
    (the bench's split and pivots per config), max shard device time (CUDA events, L2 flushed before
    each step) against the one-GPU join; the data path has no collective to leave out."""
    out = {"method": "each of W shards in turn on this GPU; projected W-GPU time = max shard device time "
                     "(broadcast / count all-reduce excluded); efficiency = t1 / (W tW)", "workloads": {}}

    def timed(j, Et, Rt, eps):
        j.run(Et, Rt, 2, eps)
        ts = []
        for _ in range(steps):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            j.run(Et, Rt, 2, eps)
            b.record(stream)
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b))
        return statistics.mean(ts)

    for name in names:
        hit = DEFAULT_HIT[name]
        eps = float(thresholds[name][f"L2@{hit:g}"]["theta"])
        E_h, Rel_h = generate_config(name)
        Et, Rt = torch.from_numpy(E_h).to(dev), torch.from_numpy(Rel_h).to(dev)
        piv, split = BEST_PIVOTS.get(name, 1), BEST_SPLIT.get(name, 0)
        with kgc.Join(device=dev.index, pivots=piv, stream=stream.cuda_stream) as j:
            t1 = timed(j, Et, Rt, eps)
        w = {"split": split, "pivots": piv, "hit_rate": hit, "ms": {"1": t1}, "shard_ms": {}, "efficiency": {}}
        for W in Ws:
            sh = []
            for rank in range(W):
                with kgc.Join(device=dev.index, pivots=piv, rank=rank, world=W, split=split,
                              stream=stream.cuda_stream) as j:
                    sh.append(timed(j, Et, Rt, eps))
            w["ms"][str(W)] = max(sh)
            w["shard_ms"][str(W)] = sh
            w["efficiency"][str(W)] = t1 / (W * max(sh))
        out["workloads"][name] = w
        del Et, Rt
    return out


def relaunch_distributed(args_argv, n):
    """--gpus N without a launcher: re-execute this script under torch.distributed.run
    (one process per GPU on this node, rendezvous on 127.0.0.1)."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *args_argv]
    return subprocess.call(cmd)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="c4", choices=sorted(CONFIGS))
    ap.add_argument("--hit", type=float, default=None, help="target hit rate of theta (default: per config)")
    ap.add_argument("--norms", default=None, help="norms joined per step, e.g. '2,1' or '2' (default: per config)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the c2 step / c3 sweep extra workloads")
    ap.add_argument("--extra-steps", type=int, default=5)
    ap.add_argument("--no-scaling", action="store_true",
                    help="skip the projected 2/4/8-GPU shard timings (c4, c5) of the N=1 line")
    ap.add_argument("--sequential", action="store_true", help="run the step's joins one after the other")
    ap.add_argument("--tail-shard", type=int, default=0,
                    help="world > 1: 1 = partition-based join (rank k holds tails [kN/W, (k+1)N/W), every query)")
    ap.add_argument("--split", default="auto",
                    help="world > 1: 0 = rank-local split, 1 = global cost-balanced, 2 = cyclic, 3 = spatial "
                         "block-cyclic heads; auto = best measured per config (c2: 2, its hits concentrate in a "
                         "few relations; c3 / c4 / c5: 3, DESIGN.md §8)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--ref-rows", type=int, default=None, help="(h,r) rows per reference step")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="diagnostic: on ONE GPU run each of W shards in turn and print the per-shard device times "
                         "(projects the N=W device time; not the official line)")
    ap.add_argument("--pivots", default="auto",
                    help="1 = the paper's single pivot; 2..8, 12, 16, 24, 32 (48, 64, 96, 128: L2 only) = multi-pivot pruning; "
                         "auto = best measured per config")
    args = ap.parse_args(argv)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and not args.emulate_ranks:
        return relaunch_distributed(argv, args.gpus)
    args.norms = [int(x) for x in (args.norms or DEFAULT_NORMS[args.config]).split(",")]
    args.hit = DEFAULT_HIT[args.config] if args.hit is None else args.hit
    args.pivots = BEST_PIVOTS.get(args.config, 1) if args.pivots == "auto" else int(args.pivots)
    args.split = BEST_SPLIT.get(args.config, 0) if args.split == "auto" else int(args.split)
    if args.ref_rows is None:
        args.ref_rows = 64 if CONFIGS[args.config].N > 100000 else 256
    cfg = CONFIGS[args.config]
    thresholds = load_thresholds()
    if args.impl == "reference":
        return run_reference(args, cfg, thresholds)
    if args.emulate_ranks:
        return run_emulated_ranks(args, cfg, thresholds)
    return run_ours(args, cfg, thresholds)


if __name__ == "__main__":
    sys.exit(main())
