"""bench.py's multi-rank path end to end on the one-GPU box: two ranks
(self-launched under torch.distributed.run) share the GPU with a gloo
control plane, the exchanges go through cudaIpc-mapped peer memory; the
line must carry n_gpus 2, the weak-scaling value, the global-gate probe, the
strong-scaling leg (analytic check) and the single-process C-ABI leg.  (NCCL
cannot put two ranks on one GPU; on multi-GPU boxes the same code runs with
NCCL.)"""

from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parent.parent


def test_two_ranks_one_gpu():
    env = dict(os.environ, QSB_BENCH_SHARE_GPU="1", QSB_BENCH_BACKEND="gloo", QSB_BENCH_STRONG_QUBITS="24")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "1",
                        "--qubits", "22"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["config"]["n_qubits"] == 23
    roof = line["roofline"]
    assert roof["bound"] == "hbm" and roof["achieved"] > 0 and roof["frac"] == roof["achieved"] / roof["peak"]
    ex = line["extras"]
    assert ex["global_gates"]["peer_nvlink"]["peer_gates_per_rep"] == 1
    assert ex["strong34"]["analytic_check_ok"] is True
    assert ex["single_process_c_abi"]["p2p_swaps"]["swaps"] > 0
    assert ex["single_process_c_abi"]["peer_gates"]["peer_gates"] > 0
