"""bench.py's launch contract on the CPU: --gpus N without a launcher fails
loudly when N GPUs are not visible (never a silent n_gpus: 1 line), a
WORLD_SIZE / --gpus mismatch is refused, and under torchrun only rank 0
prints, after every rank has torn its communicators down (finish_dist)."""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _bench(*args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True, text=True,
                          env=e, timeout=300)


def test_gpus_without_devices_fails_loudly():
    r = _bench("--gpus", "2")
    assert r.returncode != 0
    assert "GPU" in r.stderr and r.stdout.strip() == ""


def test_world_size_mismatch_refused():
    r = _bench("--gpus", "4", env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert r.returncode != 0 and "WORLD_SIZE" in r.stderr


def test_reference_arm_runs_rank0_only():
    r = _bench("--impl", "reference", "--qubits", "16", "--steps", "3", "--warmup", "1")
    assert r.returncode == 0
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["e2e"]["h2d_bytes_per_step"] == 0
    assert line["cpu_baseline"]["cores"] >= 1 and line["cpu_baseline"]["kind"] in ("reference", "port")
    r1 = _bench("--impl", "reference", "--qubits", "16", "--steps", "2", "--warmup", "1",
                env={"WORLD_SIZE": "2", "RANK": "1", "LOCAL_RANK": "1"})
    assert r1.returncode == 0 and r1.stdout.strip() == ""


FINISH = r'''
import os, sys, time
sys.path.insert(0, {root!r})
import torch.distributed as dist
dist.init_process_group("gloo")
import bench
rank = int(os.environ["RANK"])
if rank != 0:
    time.sleep(0.5)  # a slow rank: rank 0 must still print last
    print("rank%d-log-line" % rank, flush=True)
bench.finish_dist('{{"rank0": true}}' if rank == 0 else None)
'''


def test_finish_dist_rank0_prints_last(tmp_path):
    script = tmp_path / "fin.py"
    script.write_text(FINISH.format(root=str(ROOT)))
    port = 29500 + (os.getpid() % 1000)
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=3",
                        "--master-addr=127.0.0.1", f"--master-port={port}", str(script)],
                       capture_output=True, text=True, timeout=240)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert lines[-1] == '{"rank0": true}'
    assert sum(ln.startswith("rank") and "log-line" in ln for ln in lines) == 2
