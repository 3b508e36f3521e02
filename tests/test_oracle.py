"""Pin the oracle (oracle/c.py, oracle/port.py) against the reference.

Every expected value comes from tests/golden/pairsim_golden.npz, produced by
running pairsim itself (tests/golden/make_golden.py).  These tests run on the
CPU; they establish that the C restatement is bit-exact with pairsim before
any GPU result is compared against it.
"""

from __future__ import annotations

import cmath
import math

import numpy as np
import pytest

from golden_util import H_M8, X_M8, M8DGate, M8Gate, digest, golden, golden_double, hist_from_outcomes
from oracle import c as oc
from oracle import port


def replay_c(amps, ops, mats):
    for (kind, c1, c2, t), m in zip(ops, mats):
        g = M8Gate(m)
        if kind == 0:
            oc.apply_gate(amps, int(t), g)
        elif kind == 1:
            oc.apply_controlled_gate(amps, int(c1), int(t), g)
        else:
            oc.apply_cc_gate(amps, int(c1), int(c2), int(t), g)
        yield amps


class TestKnownAnswers:
    """pkg/tests/test_kernel.py:42-73"""

    def test_nth_cleared_kats(self):
        assert oc.nth_cleared(0, 0) == 0
        assert oc.nth_cleared(3, 0) == 6
        assert oc.nth_cleared(5, 1) == 9

    @pytest.mark.parametrize("n", range(1, 11))
    def test_pair_partition(self, n):
        for t in range(n):
            a = np.array([oc.nth_cleared(i, t) for i in range(1 << (n - 1))])
            union = np.sort(np.concatenate([a, a | (1 << t)]))
            assert np.array_equal(union, np.arange(1 << n))

    def test_pcg64_matches_numpy(self):
        for seed in (0, 1, 42, 2**63 + 5):
            ref = np.random.default_rng(seed).random(4099)
            got = oc.pcg64_random(seed, 4099)
            assert ref.tobytes() == got.tobytes()

    def test_hadamard_and_x(self):
        a = np.array([1, 0], np.complex64)
        oc.apply_gate(a, 0, M8Gate(H_M8))
        assert np.array_equal(a, np.full(2, np.float32(1 / math.sqrt(2)), np.complex64))
        b = np.array([1, 0, 0, 0], np.complex64)
        oc.apply_gate(b, 1, M8Gate(X_M8))
        assert np.array_equal(b, [0, 0, 1, 0])


class TestTracesBitExact:
    @pytest.mark.parametrize("n", [1, 2, 3, 5, 6, 7, 8, 10])
    def test_c_oracle_every_op(self, n):
        g = golden()
        states = g[f"trace{n}_states"]
        amps = states[0].copy()
        for k, cur in enumerate(replay_c(amps, g[f"trace{n}_ops"], g[f"trace{n}_mats"])):
            assert cur.tobytes() == states[k + 1].tobytes(), f"op {k}"

    @pytest.mark.parametrize("n", [12, 14])
    def test_c_oracle_big_digest(self, n):
        g = golden()
        amps = g[f"tracebig{n}_in"].copy()
        for _ in replay_c(amps, g[f"tracebig{n}_ops"], g[f"tracebig{n}_mats"]):
            pass
        assert digest(amps) == g["meta"][f"tracebig{n}_final"]

    @pytest.mark.parametrize("n", [5, 8, 10])
    def test_numpy_port_every_op(self, n):
        g = golden()
        states = g[f"trace{n}_states"]
        amps = states[0].copy()
        ex = port.Executor(workers=4, min_parallel_items=1)
        for k, ((kind, c1, _c2, t), m) in enumerate(zip(g[f"trace{n}_ops"], g[f"trace{n}_mats"])):
            if kind == 0:
                port.apply_gate(amps, int(t), M8Gate(m), ex)
            else:
                port.apply_controlled_gate(amps, int(c1), int(t), M8Gate(m), ex)
            assert amps.tobytes() == states[k + 1].tobytes()
        ex.close()

    @pytest.mark.parametrize("idx", range(6))
    def test_random_circuits(self, idx):
        g = golden()
        n = int(g[f"rc{idx}_n"])
        amps = np.zeros(1 << n, np.complex64)
        amps[0] = 1
        for _ in replay_c(amps, g[f"rc{idx}_ops"], g[f"rc{idx}_mats"]):
            pass
        assert amps.tobytes() == g[f"rc{idx}_final"].tobytes()


def qft_ops(n):
    """build_qft (pkg/src/pairsim/circuits.py:195-210) as (ops, mats)."""
    ops, mats = [], []
    for j in range(n):
        for k in range(j):
            d = np.complex64(cmath.exp(1j * (math.pi / 2 ** (j - k))))  # gates.py:84-86
            ops.append((1, j, -1, k))
            mats.append(np.array([1, 0, 0, 0, 0, 0, d.real, d.imag], np.float32))
        ops.append((0, -1, -1, j))
        mats.append(H_M8)
    return np.array(ops), np.array(mats, np.float32)


def basis_state(n, x):
    a = np.zeros(1 << n, np.complex64)  # X gates on |0> give exactly e_x
    a[x] = 1
    return a


class TestQftAndConfigs:
    @pytest.mark.parametrize("n", [6, 10])
    def test_qft_basis_small(self, n):
        g = golden()
        amps = basis_state(n, int(g[f"qft{n}_basis_x"]))
        ops, mats = qft_ops(n)
        for _ in replay_c(amps, ops, mats):
            pass
        assert amps.tobytes() == g[f"qft{n}_basis"].tobytes()

    @pytest.mark.parametrize("n", [16])
    def test_qft_basis_digest(self, n):
        g = golden()
        amps = basis_state(n, int(g[f"qft{n}_basis_x"]))
        ops, mats = qft_ops(n)
        for _ in replay_c(amps, ops, mats):
            pass
        assert digest(amps) == g["meta"][f"qft{n}_basis"]

    def test_hlayer12_probabilities(self):
        g = golden()
        amps = np.zeros(1 << 12, np.complex64)
        amps[0] = 1
        for q in range(12):
            oc.apply_gate(amps, q, M8Gate(H_M8))
        assert amps.tobytes() == g["hlayer12_amps"].tobytes()
        p = oc.probabilities(amps)
        assert p.tobytes() == g["hlayer12_probs"].tobytes()
        assert p.tobytes() == port.probabilities(amps).tobytes()


class TestSampling:
    @pytest.mark.parametrize("name", ["rand10", "rand16", "sparse3", "hlayer14", "decay13"])
    @pytest.mark.parametrize("seed", [0, 7, 12345])
    def test_sample_histograms(self, name, seed):
        g = golden()
        amps = g[f"samp_{name}_amps"]
        keys, counts = hist_from_outcomes(oc.sample_outcomes(amps, 5000, seed))
        assert np.array_equal(keys, g[f"samp_{name}_s{seed}_keys"])
        assert np.array_equal(counts, g[f"samp_{name}_s{seed}_counts"])
        pk, pc = hist_from_outcomes(port.sample_outcomes(amps, 5000, seed))
        assert np.array_equal(pk, keys) and np.array_equal(pc, counts)

    @pytest.mark.parametrize("name", ["rand10", "sparse3", "decay13"])
    def test_collapse_outcomes(self, name):
        g = golden()
        amps = g[f"samp_{name}_amps"]
        got = [int(oc.sample_outcomes(amps, 1, seed)[0]) for seed in range(20)]
        assert got == g[f"samp_{name}_collapse"].tolist()

    def test_degenerate(self):
        with pytest.raises(ZeroDivisionError):
            oc.sample_outcomes(np.zeros(4, np.complex64), 10, 0)


class TestDoublyControlled:
    @pytest.mark.parametrize("key", ["tof_012", "tof_402", "tof_130"])
    def test_cc_x_matches_toffoli_decomposition(self, key):
        """The derived CC oracle equals pairsim's own 6-CNOT Toffoli."""
        g = golden()
        c1, c2, t = (int(ch) for ch in key[4:])
        amps = g[f"{key}_in"].copy()
        oc.apply_cc_gate(amps, c1, c2, t, M8Gate(X_M8))
        np.testing.assert_allclose(amps, g[f"{key}_out"], atol=2e-6)


# ---- complex128 (Precision.DOUBLE) restatement vs pairsim DOUBLE outputs ----
def replay_c_double(amps, ops, mats):
    for (kind, c1, c2, t), m in zip(ops, mats):
        g = M8DGate(m)
        if kind == 0:
            oc.apply_gate(amps, int(t), g)
        elif kind == 1:
            oc.apply_controlled_gate(amps, int(c1), int(t), g)
        else:
            oc.apply_cc_gate(amps, int(c1), int(c2), int(t), g)
        yield amps


class TestDoublePrecision:
    """tests/golden/make_golden_double.py: the reference on complex128 registers."""

    @pytest.mark.parametrize("n", [1, 2, 3, 5, 6, 7, 8, 10])
    def test_c_oracle_every_op(self, n):
        g = golden_double()
        states = g[f"trace{n}_states"]
        assert states.dtype == np.complex128
        amps = states[0].copy()
        for k, cur in enumerate(replay_c_double(amps, g[f"trace{n}_ops"], g[f"trace{n}_mats"])):
            assert cur.tobytes() == states[k + 1].tobytes(), f"op {k}"

    @pytest.mark.parametrize("n", [12, 14])
    def test_c_oracle_big_digest(self, n):
        g = golden_double()
        amps = g[f"tracebig{n}_in"].copy()
        for _ in replay_c_double(amps, g[f"tracebig{n}_ops"], g[f"tracebig{n}_mats"]):
            pass
        assert digest(amps) == g["meta"][f"tracebig{n}_final"]

    def test_probabilities(self):
        g = golden_double()
        assert oc.probabilities(g["probs10_amps"]).tobytes() == g["probs10"].tobytes()

    @pytest.mark.parametrize("name", ["rand10", "decay13"])
    @pytest.mark.parametrize("seed", [0, 7, 12345])
    def test_sample_histograms(self, name, seed):
        g = golden_double()
        keys, counts = hist_from_outcomes(oc.sample_outcomes(g[f"samp_{name}_amps"], 5000, seed))
        assert np.array_equal(keys, g[f"samp_{name}_s{seed}_keys"])
        assert np.array_equal(counts, g[f"samp_{name}_s{seed}_counts"])

    @pytest.mark.parametrize("name", ["rand10", "decay13"])
    def test_collapse_outcomes(self, name):
        g = golden_double()
        amps = g[f"samp_{name}_amps"]
        got = [int(oc.sample_outcomes(amps, 1, seed)[0]) for seed in range(20)]
        assert got == g[f"samp_{name}_collapse"].tolist()

    @pytest.mark.parametrize("key", ["tof_012", "tof_402"])
    def test_cc_x_matches_toffoli_decomposition(self, key):
        g = golden_double()
        c1, c2, t = (int(ch) for ch in key[4:])
        amps = g[f"{key}_in"].copy()
        oc.apply_cc_gate(amps, c1, c2, t, M8DGate(np.array([0, 0, 1, 0, 1, 0, 0, 0], np.float64)))
        np.testing.assert_allclose(amps, g[f"{key}_out"], atol=1e-14)
