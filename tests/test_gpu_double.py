"""GPU parity for complex128 registers (pairsim Precision.DOUBLE; gates64.cu and
the templated measure chain) through the C ABI.

Expected values: the reference's own DOUBLE outputs (tests/golden/
pairsim_golden_double.npz) and the C oracle's complex128 restatement, which
test_oracle.py pins bit for bit against them.  Bar: bit-exact amplitudes (up
to the sign of zero), probabilities and sampled outcomes.
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from golden_util import M8DGate, digest, golden_double, hist_from_outcomes, same_values
from oracle import c as oc
from paper_1805_00988_b200 import State, build_hadamard_layer, build_qft, execute, random_unitary_gate, u1
from paper_1805_00988_b200 import pairsim as ps
from paper_1805_00988_b200.circuits import Apply, Circuit, ControlledApply, ControlledControlledApply
from paper_1805_00988_b200.gates import FIXED_GATES

pytestmark = pytest.mark.gpu


def rand_amps(n, rng):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return v / np.linalg.norm(v)


def load(n, amps):
    st = State(n, precision="double")
    st.set_amplitudes(amps)
    return st


def gate_mix(rng):
    lib = list(FIXED_GATES.values())
    r = rng.random()
    if r < 0.4:
        return random_unitary_gate(rng)
    if r < 0.55:
        return u1(float(rng.uniform(0, 2 * math.pi)))
    return lib[int(rng.integers(len(lib)))]


def replay(st, ops, mats):
    for (kind, c1, c2, t), m in zip(ops, mats):
        g = M8DGate(m)
        if kind == 0:
            st.apply_gate(g, int(t))
        elif kind == 1:
            st.apply_controlled_gate(g, int(c1), int(t))
        else:
            st.apply_controlled_controlled_gate(g, int(c1), int(c2), int(t))
        yield st


class TestGoldenDouble:
    @pytest.mark.parametrize("n", [1, 2, 3, 5, 6, 7, 8, 10])
    def test_every_op(self, n):
        g = golden_double()
        states = g[f"trace{n}_states"]
        st = load(n, states[0])
        assert st.amplitudes().dtype == np.complex128
        for k, cur in enumerate(replay(st, g[f"trace{n}_ops"], g[f"trace{n}_mats"])):
            assert same_values(cur.amplitudes(), states[k + 1]), f"op {k}"

    @pytest.mark.parametrize("n", [12, 14])
    def test_big_digest(self, n):
        g = golden_double()
        st = load(n, g[f"tracebig{n}_in"])
        for _ in replay(st, g[f"tracebig{n}_ops"], g[f"tracebig{n}_mats"]):
            pass
        assert digest(st.amplitudes()) == g["meta"][f"tracebig{n}_final"]

    @pytest.mark.parametrize("fuse", [False, True])
    @pytest.mark.parametrize("n", [6, 10])
    def test_qft(self, n, fuse):
        g = golden_double()
        st = State(n, precision="double").reset(int(g[f"qft{n}_basis_x"]))
        execute(build_qft(n), st, fuse=fuse)
        assert same_values(st.amplitudes(), g[f"qft{n}_basis"])
        st = State(n, precision="double")
        for q in range(n):
            st.h(q)
            st.t(q)
        for q in range(n - 1):
            st.cx(q, q + 1)
        execute(build_qft(n), st, fuse=fuse)
        assert same_values(st.amplitudes(), g[f"qft{n}_ent"])

    def test_qft16_digest(self):
        g = golden_double()
        st = State(16, precision="double").reset(int(g["qft16_basis_x"]))
        execute(build_qft(16), st)
        assert digest(st.amplitudes()) == g["meta"]["qft16_basis"]

    def test_probabilities(self):
        g = golden_double()
        st = load(10, g["probs10_amps"])
        assert st.probabilities().tobytes() == g["probs10"].tobytes()

    @pytest.mark.parametrize("name", ["rand10", "decay13"])
    @pytest.mark.parametrize("seed", [0, 7, 12345])
    def test_sample_histograms(self, name, seed):
        g = golden_double()
        amps = g[f"samp_{name}_amps"]
        st = load(int(amps.size).bit_length() - 1, amps)
        keys, counts = hist_from_outcomes(st.sample_outcomes(5000, seed))
        assert np.array_equal(keys, g[f"samp_{name}_s{seed}_keys"])
        assert np.array_equal(counts, g[f"samp_{name}_s{seed}_counts"])

    @pytest.mark.parametrize("name", ["rand10", "decay13"])
    def test_collapse(self, name):
        g = golden_double()
        amps = g[f"samp_{name}_amps"]
        n = int(amps.size).bit_length() - 1
        got = []
        for seed in range(20):
            st = load(n, amps)
            m = st.measure_collapse(seed)
            got.append(m)
            a = st.amplitudes()
            assert a[m] == 1.0 and np.count_nonzero(a) == 1
        assert got == g[f"samp_{name}_collapse"].tolist()


class TestOracleDouble:
    @pytest.mark.parametrize("n", [6, 7, 9, 13, 17])
    def test_every_target_and_control_class(self, n):
        """Lane-bit and row-bit targets and controls (shuffle / two-stream /
        phase / scalar paths), single and double controls, vs the C oracle."""
        rng = np.random.default_rng(900 + n)
        ref = rand_amps(n, rng)
        st = load(n, ref)
        for t in range(n):
            for _ in range(2):
                g = gate_mix(rng)
                r = rng.random()
                others = [q for q in range(n) if q != t]
                if r < 0.4 or n < 3:
                    st.apply_gate(g, t)
                    oc.apply_gate(ref, t, g)
                elif r < 0.8:
                    c = int(rng.choice(others))
                    st.apply_controlled_gate(g, c, t)
                    oc.apply_controlled_gate(ref, c, t, g)
                else:
                    c1, c2 = (int(x) for x in rng.choice(others, 2, replace=False))
                    st.apply_controlled_controlled_gate(g, c1, c2, t)
                    oc.apply_cc_gate(ref, c1, c2, t, g)
        assert same_values(st.amplitudes(), ref)
        assert st.probabilities().tobytes() == oc.probabilities(ref).tobytes()
        assert np.array_equal(st.sample_outcomes(3000, 5), oc.sample_outcomes(ref, 3000, 5))

    @pytest.mark.parametrize("n", [5, 11, 12, 15])
    def test_fused_equals_unfused(self, n):
        """k_small_d (n <= 12) and the per-op path (n > 12) apply circuits exactly
        as the individual sweeps do."""
        rng = np.random.default_rng(950 + n)
        a0 = rand_amps(n, rng)
        ins = []
        for _ in range(60):
            t = int(rng.integers(n))
            others = [q for q in range(n) if q != t]
            r = rng.random()
            if r < 0.5:
                ins.append(Apply(gate_mix(rng), t))
            elif r < 0.85:
                ins.append(ControlledApply(gate_mix(rng), int(rng.choice(others)), t))
            elif n >= 3:
                c1, c2 = (int(x) for x in rng.choice(others, 2, replace=False))
                ins.append(ControlledControlledApply(gate_mix(rng), c1, c2, t))
        circ = Circuit(n, tuple(ins))
        outs = []
        for fuse in (False, True):
            st = load(n, a0)
            execute(circ, st, fuse=fuse)
            outs.append(st.amplitudes())
        assert same_values(outs[0], outs[1])

    def test_swap_qubits(self):
        rng = np.random.default_rng(3)
        a = rand_amps(9, rng)
        st = load(9, a)
        st.swap_qubits(2, 7)
        idx = np.arange(1 << 9)
        b2, b7 = (idx >> 2) & 1, (idx >> 7) & 1
        perm = idx ^ ((b2 ^ b7) << 2) ^ ((b2 ^ b7) << 7)
        assert np.array_equal(st.amplitudes(), a[perm])


class TestLargeDouble:
    def test_hlayer_28_uniform(self):
        """4 GiB complex128 register: H on every qubit gives 2^-14 exactly."""
        n = 28
        st = State(n, precision="double")
        execute(build_hadamard_layer(n), st, fuse=False)
        ref = State(10, precision="double")
        execute(build_hadamard_layer(10), ref, fuse=False)
        a = st.amplitudes(0, 4096)
        assert np.all(a == a[0]) and abs(a[0].real - 2.0 ** -14) < 1e-15
        assert abs(st.norm_squared() - 1.0) < 1e-12
        st.close()


class TestPairsimShimDouble:
    """The reference's DOUBLE acceptance criteria (pkg/tests/test_acceptance.py:71-83)
    run through the shim: < 1e-10 vs a dense fp64 oracle."""

    @pytest.mark.parametrize("n", [4, 8])
    def test_vs_dense_oracle(self, n):
        rng = np.random.default_rng(n)
        sv = ps.new_state(n, ps.Precision.DOUBLE)
        assert sv.precision is ps.Precision.DOUBLE and sv.amps.dtype == np.complex128
        dense = np.zeros(1 << n, np.complex128)
        dense[0] = 1
        idx = np.arange(1 << n)
        for _ in range(40):
            g = random_unitary_gate(rng)
            t = int(rng.integers(n))
            c = int(rng.integers(n))
            U = np.array([[g.a, g.b], [g.c, g.d]], np.complex128)
            a = idx[((idx >> t) & 1) == 0]
            if c != t and rng.random() < 0.5:
                ps.apply_controlled_gate(sv, c, t, g)
                a = a[((a >> c) & 1) == 1]
            else:
                ps.apply_gate(sv, t, g)
            b = a | (1 << t)
            va, vb = dense[a].copy(), dense[b].copy()
            dense[a] = U[0, 0] * va + U[0, 1] * vb
            dense[b] = U[1, 0] * va + U[1, 1] * vb
        assert np.max(np.abs(sv.amps - dense)) < 1e-10
        assert abs(ps.norm_squared(sv) - 1.0) < 1e-10
        p = ps.probabilities(sv)
        assert np.max(np.abs(p - np.abs(dense) ** 2)) < 1e-10


class TestFusedTilesDouble:
    """complex128 fused passes as compiled TMA tile programs (fused_dev.cuh
    with 16-B one-amplitude units) against the sweeps, bit for bit."""

    @pytest.mark.parametrize("n,kind", [(14, "mixed"), (17, "qft"), (20, "layered"), (22, "hlayer")])
    def test_compiled_tiles_equal_sweeps(self, n, kind):
        import os

        from paper_1805_00988_b200 import build_hadamard_layer, layered_random_circuit

        rng = np.random.default_rng(1300 + n)
        a0 = rand_amps(n, rng)
        if kind == "mixed":
            ins = []
            for _ in range(80):
                t = int(rng.integers(n))
                others = [q for q in range(n) if q != t]
                r = rng.random()
                if r < 0.5:
                    ins.append(Apply(gate_mix(rng), t))
                elif r < 0.85:
                    ins.append(ControlledApply(gate_mix(rng), int(rng.choice(others)), t))
                else:
                    c1, c2 = (int(x) for x in rng.choice(others, 2, replace=False))
                    ins.append(ControlledControlledApply(gate_mix(rng), c1, c2, t))
            circ = Circuit(n, tuple(ins))
        else:
            circ = {"qft": build_qft(n), "layered": layered_random_circuit(n, 3, seed=n),
                    "hlayer": build_hadamard_layer(n)}[kind]
        ref = load(n, a0)
        execute(circ, ref, fuse=False)
        old = os.environ.get("QSB_FUSED_JIT")
        os.environ["QSB_FUSED_JIT"] = "2"
        try:
            st = load(n, a0)
            execute(circ, st, fuse=True)
        finally:
            if old is None:
                os.environ.pop("QSB_FUSED_JIT", None)
            else:
                os.environ["QSB_FUSED_JIT"] = old
        assert same_values(st.amplitudes(), ref.amplitudes())
