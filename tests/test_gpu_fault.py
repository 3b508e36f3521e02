"""The parity suite can fail (SURVEY 5 fault injection; the sign-flipped `c`
pattern of pkg/tests/test_cli.py:151-160): with QSB_FAULT_FLIP_C=1 the
library negates the c entry of every pair gate in the sweep and fused paths,
and the bit-exact parity tests must catch it; without the flag the same
tests pass."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parent.parent
SELECT = ["tests/test_gpu_parity.py::TestSweeps::test_every_target",
          "tests/test_gpu_parity.py::TestFusedEqualsUnfused::test_gate_classes_vs_oracle",
          "tests/test_gpu_parity.py::TestConfigs::test_qft_small_exact"]


def _run(flag: bool):
    env = dict(os.environ)
    env.pop("QSB_FAULT_FLIP_C", None)
    if flag:
        env["QSB_FAULT_FLIP_C"] = "1"
    return subprocess.run([sys.executable, "-m", "pytest", "-q", "-p", "no:cacheprovider", *SELECT],
                          cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)


def test_flipped_c_is_caught():
    r = _run(True)
    assert r.returncode != 0, r.stdout[-2000:]
    assert "failed" in r.stdout


def test_same_tests_pass_without_the_fault():
    r = _run(False)
    assert r.returncode == 0, r.stdout[-3000:]
