"""GPU parity: libqsb200 (through the C ABI) vs the oracle and the reference's
golden vectors.

Bar: bit-exact values for every amplitude (x == y elementwise; the sign of a
zero amplitude is the only freedom) and bit-exact fp64
probabilities / sampled outcomes.  The north_star tolerance (rtol 1e-5) is
therefore met with margin; size-independent properties cover n = 28..30.
"""

from __future__ import annotations

import json
import math
import os
from contextlib import contextmanager
from pathlib import Path

import numpy as np
import pytest

from golden_util import H_M8, X_M8, M8Gate, digest, golden, hist_from_outcomes, same_values
from oracle import c as oc
from paper_1805_00988_b200 import (
    FIXED_GATES,
    CapacityError,
    DegenerateStateError,
    State,
    build_hadamard_layer,
    build_qft,
    execute,
    layered_random_circuit,
    random_circuit,
    random_unitary_gate,
    u1,
)
from paper_1805_00988_b200.circuits import Apply, Circuit, ControlledApply, ControlledControlledApply

pytestmark = pytest.mark.gpu

LARGE = Path(__file__).resolve().parent / "golden" / "pairsim_golden_large.json"


def rand_amps(n, rng):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return (v / np.linalg.norm(v)).astype(np.complex64)


def load(n, amps):
    st = State(n)
    st.set_amplitudes(amps)
    return st


@contextmanager
def env(**kv):
    old = {k: os.environ.get(k) for k in kv}
    os.environ.update({k: str(v) for k, v in kv.items()})
    try:
        yield
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def gate_mix(rng):
    lib = list(FIXED_GATES.values())
    r = rng.random()
    if r < 0.4:
        return random_unitary_gate(rng)
    if r < 0.55:
        return u1(float(rng.uniform(0, 2 * math.pi)))
    return lib[int(rng.integers(len(lib)))]


class TestSweeps:
    @pytest.mark.parametrize("n", [1, 2, 3, 5, 6, 7, 8, 9, 11, 14, 17])
    def test_every_target(self, n):
        rng = np.random.default_rng(100 + n)
        ref = rand_amps(n, rng)
        st = load(n, ref)
        for rep in range(2):
            for t in range(n):
                g = gate_mix(rng)
                st.apply_gate(g, t)
                oc.apply_gate(ref, t, g)
                assert same_values(st.amplitudes(), ref), (rep, t)

    @pytest.mark.parametrize("n", [2, 5, 8, 9])
    def test_controlled_all_pairs(self, n):
        rng = np.random.default_rng(200 + n)
        ref = rand_amps(n, rng)
        st = load(n, ref)
        for c in range(n):
            for t in range(n):
                if c == t:
                    continue
                g = gate_mix(rng)
                st.apply_controlled_gate(g, c, t)
                oc.apply_controlled_gate(ref, c, t, g)
        assert same_values(st.amplitudes(), ref)

    @pytest.mark.parametrize("n", [12, 16])
    def test_controlled_random_pairs(self, n):
        rng = np.random.default_rng(300 + n)
        ref = rand_amps(n, rng)
        st = load(n, ref)
        for _ in range(60):
            c, t = (int(x) for x in rng.choice(n, 2, replace=False))
            g = gate_mix(rng)
            st.apply_controlled_gate(g, c, t)
            oc.apply_controlled_gate(ref, c, t, g)
        assert same_values(st.amplitudes(), ref)

    @pytest.mark.parametrize("n", [3, 7, 10, 15])
    def test_doubly_controlled(self, n):
        rng = np.random.default_rng(400 + n)
        ref = rand_amps(n, rng)
        st = load(n, ref)
        for _ in range(40):
            c1, c2, t = (int(x) for x in rng.choice(n, 3, replace=False))
            g = gate_mix(rng)
            st.apply_controlled_controlled_gate(g, c1, c2, t)
            oc.apply_cc_gate(ref, c1, c2, t, g)
        assert same_values(st.amplitudes(), ref)

    @pytest.mark.parametrize("knob", [{"QSB_FORCE_SCALAR": 1}, {"QSB_SWEEP_U": 1}, {"QSB_SWEEP_U": 4},
                                      {"QSB_NO_PHASE": 1}, {"QSB_BLOCKS_PER_SM": 1}])
    def test_kernel_variants_bit_identical(self, knob):
        n = 13
        rng = np.random.default_rng(7)
        a0 = rand_amps(n, rng)
        ops = [(gate_mix(rng), int(rng.integers(n)), int(rng.integers(n))) for _ in range(50)]
        outs = []
        for kv in ({}, knob):
            with env(**kv):
                st = load(n, a0)
                for g, c, t in ops:
                    if c == t:
                        st.apply_gate(g, t)
                    else:
                        st.apply_controlled_gate(g, c, t)
                outs.append(st.amplitudes())
        assert same_values(outs[0], outs[1])


class TestGoldenTraces:
    @pytest.mark.parametrize("n", [1, 2, 3, 5, 6, 7, 8, 10])
    def test_every_op(self, n):
        g = golden()
        states = g[f"trace{n}_states"]
        st = load(n, states[0])
        for k, ((kind, c, _c2, t), m) in enumerate(zip(g[f"trace{n}_ops"], g[f"trace{n}_mats"])):
            if kind == 0:
                st.apply_gate(M8Gate(m), int(t))
            else:
                st.apply_controlled_gate(M8Gate(m), int(c), int(t))
            assert same_values(st.amplitudes(), states[k + 1]), k

    @pytest.mark.parametrize("n", [12, 14])
    def test_big_trace_digest(self, n):
        g = golden()
        st = load(n, g[f"tracebig{n}_in"])
        for (kind, c, _c2, t), m in zip(g[f"tracebig{n}_ops"], g[f"tracebig{n}_mats"]):
            if kind == 0:
                st.apply_gate(M8Gate(m), int(t))
            else:
                st.apply_controlled_gate(M8Gate(m), int(c), int(t))
        assert digest(st.amplitudes()) == g["meta"][f"tracebig{n}_final"]

    @pytest.mark.parametrize("idx", range(6))
    def test_pairsim_random_circuits(self, idx):
        """random_circuit here consumes the RNG like pairsim's (circuits.py:229-255)."""
        g = golden()
        rc_rng = np.random.default_rng(55)
        for _ in range(idx + 1):
            n = int(rc_rng.integers(1, 11))
            circ = random_circuit(n, int(rc_rng.integers(1, 41)), rc_rng)
        assert n == int(g[f"rc{idx}_n"])
        for fuse in (False, True):
            st = State(n)
            execute(circ, st, fuse=fuse)
            assert same_values(st.amplitudes(), g[f"rc{idx}_final"])


class TestConfigs:
    @pytest.mark.parametrize("n", [6, 10])
    @pytest.mark.parametrize("fuse", [False, True])
    def test_qft_small_exact(self, n, fuse):
        g = golden()
        st = State(n).reset(int(g[f"qft{n}_basis_x"]))
        execute(build_qft(n), st, fuse=fuse)
        assert same_values(st.amplitudes(), g[f"qft{n}_basis"])
        st = entangled(n)
        execute(build_qft(n), st, fuse=fuse)
        assert same_values(st.amplitudes(), g[f"qft{n}_ent"])

    @pytest.mark.parametrize("n", [16, 20])
    @pytest.mark.parametrize("fuse", [False, True])
    def test_qft_digest(self, n, fuse):
        g = golden()
        st = State(n).reset(int(g[f"qft{n}_basis_x"]))
        execute(build_qft(n), st, fuse=fuse)
        assert digest(st.amplitudes()) == g["meta"][f"qft{n}_basis"]
        st = entangled(n)
        execute(build_qft(n), st, fuse=fuse)
        assert digest(st.amplitudes()) == g["meta"][f"qft{n}_ent"]

    @pytest.mark.parametrize("fuse", [False, True])
    def test_config1_hlayer20_probabilities(self, fuse):
        g = golden()
        st = State(20)
        execute(build_hadamard_layer(20), st, fuse=fuse)
        assert digest(st.amplitudes()) == g["meta"]["hlayer20_amps"]
        assert digest(st.probabilities()) == g["meta"]["hlayer20_probs"]

    def test_hlayer12_probabilities_bytes(self):
        g = golden()
        st = State(12)
        for q in range(12):
            st.h(q)
        assert st.probabilities().tobytes() == g["hlayer12_probs"].tobytes()

    @pytest.mark.skipif(not LARGE.exists(), reason="large golden digests not generated")
    @pytest.mark.parametrize("fuse", [True, False])
    def test_config3_qft_large(self, fuse):
        """28-qubit QFT vs the reference CPU amplitudes (BASELINE config 3)."""
        large = json.loads(LARGE.read_text())
        for n in (24, 28):
            if f"qft{n}_basis" not in large:
                continue
            rec = large[f"qft{n}_basis"]
            st = State(n).reset(rec["x"])
            execute(build_qft(n), st, fuse=fuse)
            assert digest(st.amplitudes()) == rec["amps"], n
            assert digest(st.probabilities()) == rec["probs"], n
            st.close()
            st = entangled(n)
            execute(build_qft(n), st, fuse=fuse)
            assert digest(st.amplitudes()) == large[f"qft{n}_ent"]["amps"], n
            st.close()


def entangled(n):
    """make_golden.prep_entangled: H+T on every qubit, then a CX chain."""
    st = State(n)
    for q in range(n):
        st.h(q)
        st.t(q)
    for q in range(n - 1):
        st.cx(q, q + 1)
    return st


class TestFusedEqualsUnfused:
    @pytest.mark.parametrize("rb", ["3", "4"])
    @pytest.mark.parametrize("n,K", [(10, 10), (12, 11), (13, 13), (16, 12), (18, 13), (19, 14)])
    def test_random_circuits(self, n, K, rb):
        rng = np.random.default_rng(500 + n)
        a0 = rand_amps(n, rng)
        circ = random_circuit(n, 120, rng)
        # add doubly-controlled gates too
        extra = []
        for _ in range(10):
            c1, c2, t = (int(x) for x in rng.choice(n, 3, replace=False))
            extra.append(ControlledControlledApply(gate_mix(rng), c1, c2, t))
        circ = Circuit(n, circ.instructions + tuple(extra))
        outs = []
        with env(QSB_FUSED_RB=rb):
            for fuse in (False, True):
                st = load(n, a0)
                execute(circ, st, fuse=fuse, tile_qubits=K)
                outs.append(st.amplitudes())
        assert same_values(outs[0], outs[1])

    @pytest.mark.parametrize("rb", ["3", "4"])
    @pytest.mark.parametrize("n,K", [(13, 13), (16, 12), (17, 13)])
    def test_gate_classes_vs_oracle(self, n, K, rb):
        """Every fused gate class (complex, real, H-like, X, phase) on every
        tile target, plain and controlled, bit for bit against the oracle.
        Real rotations and scaled H-like gates are the cases where a fused
        multiply-add of two products would change the last bit."""
        rng = np.random.default_rng(700 + n + K)
        a0 = rand_amps(n, rng)

        def real_rot():
            th = float(rng.uniform(0, 2 * math.pi))
            return M8Gate(np.array([math.cos(th), 0, -math.sin(th), 0,
                                    math.sin(th), 0, math.cos(th), 0], dtype=np.float32))

        def h_like():
            a, b = (float(x) for x in rng.uniform(-1, 1, 2))
            return M8Gate(np.array([a, 0, b, 0, a, 0, -b, 0], dtype=np.float32))

        makers = [real_rot, h_like, lambda: M8Gate(H_M8), lambda: M8Gate(X_M8),
                  lambda: random_unitary_gate(rng), lambda: u1(float(rng.uniform(0, 6.28)))]
        ins = []
        tile = list(range(6)) + list(range(n - (K - 6), n))
        for rep in range(3):
            for t in tile:
                g = makers[int(rng.integers(len(makers)))]()
                r = rng.random()
                others = [q for q in range(n) if q != t]
                if r < 0.5:
                    ins.append(Apply(g, t))
                elif r < 0.85:
                    ins.append(ControlledApply(g, int(rng.choice(others)), t))
                else:
                    c1, c2 = (int(x) for x in rng.choice(others, 2, replace=False))
                    ins.append(ControlledControlledApply(g, c1, c2, t))
        circ = Circuit(n, tuple(ins))
        ref = a0.copy()
        for i in circ.instructions:
            if isinstance(i, Apply):
                oc.apply_gate(ref, i.target, i.gate)
            elif isinstance(i, ControlledApply):
                oc.apply_controlled_gate(ref, i.control, i.target, i.gate)
            else:
                oc.apply_cc_gate(ref, i.control1, i.control2, i.target, i.gate)
        with env(QSB_FUSED_RB=rb):
            st = load(n, a0)
            execute(circ, st, fuse=True, tile_qubits=K)
            assert same_values(st.amplitudes(), ref)

    @pytest.mark.parametrize("n", [1, 2, 3, 5, 8, 9, 12, 13])
    def test_small_register_single_launch(self, n):
        """n < 10 fused passes run in one shared-memory launch (k_small)."""
        rng = np.random.default_rng(600 + n)
        a0 = rand_amps(n, rng)
        circ = random_circuit(n, 150, rng)
        if n >= 3:
            extra = []
            for _ in range(10):
                c1, c2, t = (int(x) for x in rng.choice(n, 3, replace=False))
                extra.append(ControlledControlledApply(gate_mix(rng), c1, c2, t))
            circ = Circuit(n, circ.instructions + tuple(extra))
        ref = a0.copy()
        for ins in circ.instructions:
            if isinstance(ins, Apply):
                oc.apply_gate(ref, ins.target, ins.gate)
            elif isinstance(ins, ControlledApply):
                oc.apply_controlled_gate(ref, ins.control, ins.target, ins.gate)
            else:
                oc.apply_cc_gate(ref, ins.control1, ins.control2, ins.target, ins.gate)
        st = load(n, a0)
        execute(circ, st, fuse=True, tile_qubits=n)
        assert same_values(st.amplitudes(), ref)

    def test_register_cache_reuse(self):
        """Destroyed registers park their buffers; a new one starts at |0>."""
        for _ in range(3):
            st = State(18)
            st.h(3)
            st.close()
        st = State(18)
        assert st.amplitude(0) == 1 and st.norm_squared() == 1.0
        assert np.count_nonzero(st.amplitudes()) == 1

    def test_layered_config4_shape(self):
        n = 20
        circ = layered_random_circuit(n, 6, seed=32)
        outs = []
        for fuse in (False, True):
            st = State(n)
            execute(circ, st, fuse=fuse)
            outs.append(st.amplitudes())
        assert same_values(outs[0], outs[1])
        ref = np.zeros(1 << n, np.complex64)
        ref[0] = 1
        for ins in circ.instructions:
            if isinstance(ins, Apply):
                oc.apply_gate(ref, ins.target, ins.gate)
            else:
                oc.apply_controlled_gate(ref, ins.control, ins.target, ins.gate)
        assert same_values(outs[1], ref)


class TestMeasurement:
    @pytest.mark.parametrize("name", ["rand10", "rand16", "sparse3", "hlayer14", "decay13"])
    @pytest.mark.parametrize("seed", [0, 7, 12345])
    def test_sample_histograms(self, name, seed):
        g = golden()
        amps = g[f"samp_{name}_amps"]
        n = int(amps.size).bit_length() - 1
        st = load(n, amps)
        keys, counts = hist_from_outcomes(st.sample_outcomes(5000, seed))
        assert np.array_equal(keys, g[f"samp_{name}_s{seed}_keys"])
        assert np.array_equal(counts, g[f"samp_{name}_s{seed}_counts"])

    @pytest.mark.parametrize("name", ["rand10", "rand16", "sparse3", "hlayer14", "decay13"])
    def test_collapse(self, name):
        g = golden()
        amps = g[f"samp_{name}_amps"]
        n = int(amps.size).bit_length() - 1
        for seed in range(20):
            st = load(n, amps)
            m = st.measure_collapse(seed)
            assert m == g[f"samp_{name}_collapse"][seed]
            out = st.amplitudes()
            assert out[m] == 1 and np.count_nonzero(out) == 1

    def test_per_draw_outcomes_match_oracle(self):
        rng = np.random.default_rng(3)
        for n in (1, 4, 12, 13, 18):
            amps = rand_amps(n, rng)
            st = load(n, amps)
            for seed in (0, 99):
                assert np.array_equal(st.sample_outcomes(3000, seed), oc.sample_outcomes(amps, 3000, seed))

    def test_hlayer20_histogram_digest(self):
        g = golden()
        st = State(20)
        for q in range(20):
            st.h(q)
        keys, counts = hist_from_outcomes(st.sample_outcomes(100_000, 2026))
        assert digest(np.stack([keys, counts])) == g["meta"]["samp_hlayer20_s2026"]

    def test_bernstein_vazirani_14(self):
        g = golden()
        st = State(14)
        for q in range(14):
            st.h(q)
        for q in range(14):
            if (101 >> q) & 1:
                st.z(q)
        for q in range(14):
            st.h(q)
        assert st.measure(1000, seed=20260808) == dict(zip(g["bv14_keys"].tolist(), g["bv14_counts"].tolist()))

    def test_degenerate(self):
        st = State(3)
        st.set_amplitudes(np.zeros(8, np.complex64))
        with pytest.raises(DegenerateStateError):
            st.sample_outcomes(10, 0)
        with pytest.raises(DegenerateStateError):
            st.measure_collapse(0)

    def test_probabilities_bit_exact_random(self):
        rng = np.random.default_rng(8)
        for n in (1, 9, 17):
            amps = rand_amps(n, rng)
            st = load(n, amps)
            assert st.probabilities().tobytes() == oc.probabilities(amps).tobytes()
            assert abs(st.norm_squared() - float(oc.probabilities(amps).sum())) < 1e-12

    def test_wide_dynamic_range_sampling(self):
        """Probabilities spanning ~60 binades: the binade-crossing slow path."""
        n = 16
        w = np.exp(-np.arange(1 << n) / 400.0) * np.exp(0.5j * np.arange(1 << n))
        amps = (w / np.linalg.norm(w)).astype(np.complex64)
        st = load(n, amps)
        for seed in (1, 2, 3):
            assert np.array_equal(st.sample_outcomes(20000, seed), oc.sample_outcomes(amps, 20000, seed))


class TestToffoli:
    @pytest.mark.parametrize("key", ["tof_012", "tof_402", "tof_130"])
    def test_ccx_vs_pairsim_decomposition(self, key):
        g = golden()
        c1, c2, t = (int(ch) for ch in key[4:])
        st = load(5, g[f"{key}_in"])
        st.ccx(c1, c2, t)
        np.testing.assert_allclose(st.amplitudes(), g[f"{key}_out"], atol=2e-6)


class TestErrors:
    def test_conventions(self):
        st = State(3)
        with pytest.raises(IndexError):
            st.h(3)
        with pytest.raises(IndexError):
            st.cx(-1, 0)
        with pytest.raises(ValueError):
            st.cx(1, 1)
        with pytest.raises(ValueError):
            st.ccx(0, 0, 1)
        with pytest.raises(IndexError):
            st.amplitude(8)
        with pytest.raises(ValueError):
            State(0)
        with pytest.raises(ValueError):
            st.sample_outcomes(0)

    def test_capacity_before_allocation(self):
        with pytest.raises(CapacityError) as e:
            State(30, memory_budget=8_000_000_000)
        assert "8589934592" in str(e.value)
        st = State(20, memory_budget=8 << 20)  # equal to the need: allowed
        assert st.amplitude(0) == 1
        with pytest.raises(CapacityError):
            State(40)


class TestLargeRegisters:
    """Size-independent properties at BASELINE's full sizes."""

    def test_hlayer30_uniform(self):
        n = 30
        st = State(n)
        for q in range(n):
            st.h(q)
        v = np.float32(1.0)
        h = np.float32(1 / math.sqrt(2))
        for _ in range(n):
            v = np.float32(h * v)
        step = 1 << 26
        for off in range(0, 1 << n, step):
            a = st.amplitudes(off, step)
            assert np.all(a.real == v) and np.all(a.imag == 0), off
        assert abs(st.norm_squared() - float(v) ** 2 * 2.0 ** n) < 1e-9

    def test_round_trip_every_target_n28(self):
        n = 28
        rng = np.random.default_rng(28)
        st = State(n)
        for q in range(n):
            st.h(q)
            st.t(q)
        before = st.amplitudes(0, 1 << 20)
        g = random_unitary_gate(rng)
        for t in range(n):
            st.apply_gate(g, t)
            st.apply_gate(g.dagger(), t)
        after = st.amplitudes(0, 1 << 20)
        assert np.max(np.abs(after - before)) < 1e-5 * np.max(np.abs(before)) * 10
        assert abs(st.norm_squared() - 1.0) < 1e-4

    def test_qft_analytic_n26(self):
        """QFT|x>[k] = exp(2 pi i k rev(x) / N) / sqrt(N) (no trailing swaps)."""
        n = 26
        x = 0b10110011100011110000101101
        st = State(n).reset(x)
        execute(build_qft(n), st, fuse=True)
        rev = int(format(x, f"0{n}b")[::-1], 2)
        ks = np.arange(0, 1 << n, 4099, dtype=np.int64)
        got = np.array([st.amplitude(int(k)) for k in ks[:200]])
        want = np.exp(2j * np.pi * ((ks[:200] * rev) % (1 << n)) / (1 << n)) / math.sqrt(1 << n)
        assert np.max(np.abs(got - want)) < 1e-4 * abs(want[0])


class TestGraphs:
    """Recorded gate sequences (CUDA graphs, qs_begin_capture / qs_graph_launch)
    replay with the same bits as running the gates again."""

    @pytest.mark.parametrize("n,fuse", [(8, True), (12, False), (16, True), (16, False)])
    def test_replay_equals_rerun(self, n, fuse):
        rng = np.random.default_rng(4000 + n)
        a0 = rand_amps(n, rng)
        circ = Circuit(n, build_hadamard_layer(n).instructions + random_circuit(n, 40, rng).instructions
                       + build_qft(n).instructions)
        ref = load(n, a0)
        for _ in range(3):
            execute(circ, ref, fuse=fuse)
        st = load(n, a0)
        execute(circ, st, fuse=fuse)  # first run (queues pass programs)
        with st.record() as rec:
            execute(circ, st, fuse=fuse)
        rec.graph.replay(1)  # the recorded block has not run yet: this is run 2
        rec.graph.replay(1)
        assert same_values(st.amplitudes(), ref.amplitudes())
        rec.graph.close()

    def test_getters_fail_while_recording(self):
        st = State(6)
        with pytest.raises(Exception):
            with st.record():
                st.h(0)
                st.amplitudes()
        st.h(1)  # the handle is usable again
        assert st.amplitudes().shape == (64,)
