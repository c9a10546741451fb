"""Summarise ncu output of a bench run into profiles/ (tracked).

usage: python scripts/ncu_summary.py TAG [--workload c2]
  reads gpurun_out/launches_TAG.csv   (ncu --metrics gpu__time_duration.sum launch list)
        gpurun_out/prof_TAG.ncu-rep   (ncu --set full capture of the tile / verify kernels)
  writes profiles/TAG_launches.md, profiles/TAG_ncu_full.md, profiles/TAG_launches.csv
  and updates profiles/ncu_traffic.json (dram bytes per launch per kernel, read by bench.py)
"""
import csv
import io
import json
import subprocess
import sys
from collections import OrderedDict, defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe % (elapsed)"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe % (active)"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe % (active)"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "FP64 pipe % (active)"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("smsp__inst_executed.sum", "warp instructions"),
]
UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def short(name: str) -> str:
    n = name.split("(")[0]
    for pre in ("void ", "kgc::"):
        n = n.replace(pre, "")
    return n.strip()


def launches(tag):
    p = OUT / f"launches_{tag}.csv"
    text = p.read_text()
    body = text[text.index('"ID"'):]
    rows = list(csv.DictReader(io.StringIO(body)))
    (PROF / f"{tag}_launches.csv").write_text(body)
    per = OrderedDict()
    for r in rows:
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        k = short(r["Kernel Name"])
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "nsecond": 1e-6}.get(
            r["Metric Unit"], 1e-6)
        per.setdefault(k, []).append(float(r["Metric Value"].replace(",", "")) * scale)
    total = sum(sum(v) for v in per.values())
    lines = [f"# {tag}: launch list (ncu --metrics gpu__time_duration.sum --clock-control none)", "",
             "Cold-cache, serialised per-launch device times; compare SHARES with bench.py's event times, "
             "not absolutes.  All launches of the profiled process (warm-up + timed steps, both norms).", "",
             "| kernel | launches | total ms | share |", "|---|---:|---:|---:|"]
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v):.3f} | {100 * sum(v) / total:.1f}% |")
    lines.append(f"| **total** | {sum(len(v) for v in per.values())} | {total:.3f} | 100% |")
    (PROF / f"{tag}_launches.md").write_text("\n".join(lines) + "\n")
    return per


def full(tag, workload):
    rep = OUT / f"prof_{tag}.ncu-rep"
    raw_csv = OUT / f"prof_{tag}_raw.csv"   # exported on the GPU box when the report is too large to copy
    if raw_csv.exists():
        raw = raw_csv.read_text()
    else:
        raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}
    lines = [f"# {tag}: ncu --set full --clock-control none (tile engines + verify)", "",
             f"Workload: {workload}.  Source: `gpurun_out/prof_{tag}.ncu-rep` (not tracked; regenerate with "
             "scripts/gpu_check.sh).", ""]
    traffic_path = PROF / "ncu_traffic.json"
    traffic = json.loads(traffic_path.read_text()) if traffic_path.exists() else {}
    agg = defaultdict(list)
    for r in data:
        name = short(r[col["Kernel Name"]])
        vals = {}
        for m, label in METRICS:
            if m in col:
                v = r[col[m]].replace(",", "")
                u = units[col[m]]
                try:
                    x = float(v)
                except ValueError:
                    continue
                if m.startswith("dram__bytes") or m == "lts__t_bytes.sum":
                    x *= UNIT_SCALE.get(u, 1)
                    u = "byte"
                vals[m] = (x, u)
        agg[name].append(vals)
    for name, lst in agg.items():
        lines += [f"## `{name}` ({len(lst)} launch(es) captured)", "", "| metric | " +
                  " | ".join(f"launch {i}" for i in range(len(lst))) + " |", "|---|" + "---:|" * len(lst)]
        for m, label in METRICS:
            cells = []
            for vals in lst:
                if m in vals:
                    x, u = vals[m]
                    cells.append(f"{x / 1e6:.1f} MB" if u == "byte" else f"{x:.4g} {u}")
                else:
                    cells.append("-")
            lines.append(f"| {label} (`{m}`) | " + " | ".join(cells) + " |")
        lines.append("")
        rd = [v.get("dram__bytes_read.sum", (None,))[0] for v in lst]
        wr = [v.get("dram__bytes_write.sum", (None,))[0] for v in lst]
        per_launch = [a + b for a, b in zip(rd, wr) if a is not None and b is not None]
        if per_launch:
            traffic.setdefault(workload, {})[name] = {"dram_bytes_per_launch": per_launch[-1], "tag": tag,
                                                      "all_launches": per_launch}
    (PROF / f"{tag}_ncu_full.md").write_text("\n".join(lines) + "\n")
    traffic_path.write_text(json.dumps(traffic, indent=1))


if __name__ == "__main__":
    tag = sys.argv[1]
    workload = sys.argv[sys.argv.index("--workload") + 1] if "--workload" in sys.argv else "c2"
    PROF.mkdir(exist_ok=True)
    if (OUT / f"launches_{tag}.csv").exists():
        launches(tag)
    if (OUT / f"prof_{tag}.ncu-rep").exists() or (OUT / f"prof_{tag}_raw.csv").exists():
        full(tag, workload)
    print("wrote", sorted(p.name for p in PROF.glob(f"{tag}*")))
