"""bench.py host logic on CPU (no GPU): the multi-rank launch path and the world-size check.

`bench.py --gpus N` without a launcher re-executes itself under torch.distributed.run (one
process per GPU, 127.0.0.1 rendezvous); under a launcher WORLD_SIZE must equal --gpus.  The
reference arm (the oracle, CPU only) exercises the real spawn machinery here: rank 0 prints
the one JSON line, the other ranks exit 0 without work.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def _env(**kw):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    env.update(kw)
    return env


def test_spawns_ranks_without_launcher():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--impl", "reference", "--config", "c1",
                        "--steps", "1", "--warmup", "0", "--ref-rows", "16"],
                       capture_output=True, text=True, timeout=600, env=_env(OMP_NUM_THREADS="2"), cwd=str(ROOT))
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    assert lines[0]["impl"] == "reference" and lines[0]["n_gpus"] == 2


def test_relaunch_command(monkeypatch):
    sys.path.insert(0, str(ROOT))
    import bench
    seen = {}

    def fake_call(cmd):
        seen["cmd"] = cmd
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        monkeypatch.delenv(k, raising=False)
    assert bench.main(["--gpus", "4", "--steps", "2"]) == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "--master-addr=127.0.0.1" in cmd and "--nnodes=1" in cmd
    assert cmd[-3:] == ["--gpus", "4", "--steps", "2"][-3:]


def test_world_size_mismatch_fails():
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "1", "--config", "c1"],
                       capture_output=True, text=True, timeout=600,
                       env=_env(WORLD_SIZE="2", RANK="0", LOCAL_RANK="0"), cwd=str(ROOT))
    assert r.returncode == 2
    assert "WORLD_SIZE" in r.stderr
