"""The reference's own test logic, re-pointed at the B200 backend through the
pairsim-compatible shim (paper_1805_00988_b200.pairsim).

Mirrors pkg/tests/test_kernel.py, test_measure.py, test_state.py and
test_circuits.py case by case (single precision: the device stores complex64).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import paper_1805_00988_b200.pairsim as ps

pytestmark = pytest.mark.gpu

R2 = np.float32(1 / math.sqrt(2))


def random_state(n, rng):
    st = ps.new_state(n)
    v = rng.normal(size=st.dim) + 1j * rng.normal(size=st.dim)
    st.amps[:] = (v / np.linalg.norm(v)).astype(np.complex64)
    return st


def dense_lift(gate, target, n):
    eye_hi = np.eye(1 << (n - 1 - target))
    eye_lo = np.eye(1 << target)
    return np.kron(np.kron(eye_hi, np.array([[gate.a, gate.b], [gate.c, gate.d]])), eye_lo)


def dense_controlled_lift(gate, control, target, n):
    lifted = dense_lift(gate, target, n)
    cs = ((np.arange(1 << n) >> control) & 1).astype(float)
    return np.diag(1 - cs) + lifted * cs[None, :]


class TestApplyGate:  # pkg/tests/test_kernel.py:76-121
    def test_hadamard_on_zero(self):
        st = ps.apply_gate(ps.new_state(1), 0, ps.H)
        np.testing.assert_allclose(st.amps, [R2, R2], atol=1e-7)

    def test_x_flips_bit_one(self):
        st = ps.apply_gate(ps.new_state(2), 1, ps.X)
        np.testing.assert_array_equal(st.amps, [0, 0, 1, 0])

    def test_target_out_of_range(self):
        with pytest.raises(IndexError):
            ps.apply_gate(ps.new_state(2), 2, ps.X)

    def test_matches_dense_lift(self):
        rng = np.random.default_rng(42)
        for _ in range(25):
            g = ps.random_unitary_gate(rng)
            st = random_state(6, rng)
            expected = dense_lift(g, 3, 6) @ st.amps.astype(np.complex128)
            ps.apply_gate(st, 3, g)
            assert np.abs(st.amps - expected).max() < 1e-5

    def test_unitary_round_trip(self):
        rng = np.random.default_rng(3)
        g = ps.random_unitary_gate(rng)
        st = random_state(5, rng)
        before = st.amps.copy()
        ps.apply_gate(ps.apply_gate(st, 2, g), 2, g.dagger())
        np.testing.assert_allclose(st.amps, before, atol=1e-6)

    def test_norm_preserved(self):
        rng = np.random.default_rng(9)
        st = ps.new_state(8)
        for _ in range(100):
            ps.apply_gate(st, int(rng.integers(8)), ps.random_unitary_gate(rng))
        assert abs(ps.norm_squared(st) - 1.0) < 1e-4


class TestApplyControlledGate:  # pkg/tests/test_kernel.py:124-182
    def test_cnot_truth_table(self):
        st = ps.new_state(2)
        st.amps[:] = [0, 0, 1, 0]
        ps.apply_controlled_gate(st, 1, 0, ps.X)
        np.testing.assert_array_equal(st.amps, [0, 0, 0, 1])

    def test_control_clear_is_identity(self):
        st = ps.new_state(2)
        st.amps[:] = [0, 1, 0, 0]
        ps.apply_controlled_gate(st, 1, 0, ps.X)
        np.testing.assert_array_equal(st.amps, [0, 1, 0, 0])

    def test_phase_lands_on_11_only(self):
        st = ps.new_state(2)
        st.amps[:] = 0.5
        ps.apply_controlled_gate(st, 0, 1, ps.u1(np.pi / 2))
        np.testing.assert_allclose(st.amps, [0.5, 0.5, 0.5, 0.5j], atol=1e-7)

    def test_control_equal_target(self):
        with pytest.raises(ValueError):
            ps.apply_controlled_gate(ps.new_state(2), 1, 1, ps.X)

    @pytest.mark.parametrize("bad", [-1, 5])
    def test_control_out_of_range(self, bad):
        with pytest.raises(IndexError):
            ps.apply_controlled_gate(ps.new_state(3), bad, 0, ps.X)

    def test_matches_dense_oracle(self):
        rng = np.random.default_rng(77)
        for _ in range(25):
            g = ps.random_unitary_gate(rng)
            c, t = rng.choice(6, size=2, replace=False)
            st = random_state(6, rng)
            expected = dense_controlled_lift(g, int(c), int(t), 6) @ st.amps.astype(np.complex128)
            ps.apply_controlled_gate(st, int(c), int(t), g)
            assert np.abs(st.amps - expected).max() < 1e-5

    def test_mirror_identity_kept(self):
        """A handed-out amps array stays the register's live view."""
        st = ps.new_state(3)
        view = st.amps
        ps.apply_gate(st, 0, ps.X)
        assert view is st.amps and view[1] == 1


class TestMeasure:  # pkg/tests/test_measure.py
    def test_fresh_register(self):
        np.testing.assert_array_equal(ps.probabilities(ps.new_state(3)), [1, 0, 0, 0, 0, 0, 0, 0])

    def test_scalar_recomputation(self):
        st = random_state(8, np.random.default_rng(2))
        probs = ps.probabilities(st)
        a = st.amps
        exp = a.real.astype(np.float64) ** 2 + a.imag.astype(np.float64) ** 2
        assert probs.tobytes() == exp.tobytes()

    def test_state_not_mutated(self):
        st = random_state(6, np.random.default_rng(3))
        before = st.amps.tobytes()
        ps.probabilities(st)
        ps.sample(st, 1000, seed=1)
        assert st.amps.tobytes() == before

    def test_deterministic_outcome(self):
        h = ps.sample(ps.new_state(4), 1000, seed=0)
        assert h.counts == {0: 1000} and h.samples == 1000

    def test_binomial_fair_coin(self):
        st = ps.new_state(1)
        st.amps[:] = [R2, R2]
        draws = 100_000
        h = ps.sample(st, draws, seed=99)
        assert abs(h.counts[0] / draws - 0.5) < 5 * math.sqrt(0.25 / draws)

    def test_seed_reproducibility(self):
        st = random_state(5, np.random.default_rng(7))
        assert ps.sample(st, 5000, seed=42).counts == ps.sample(st, 5000, seed=42).counts
        assert ps.sample(st, 5000, seed=42).counts != ps.sample(st, 5000, seed=43).counts

    def test_total_variation(self):
        st = random_state(2, np.random.default_rng(11))
        draws = 200_000
        h = ps.sample(st, draws, seed=5)
        emp = np.array([h.counts.get(j, 0) / draws for j in range(4)])
        assert 0.5 * np.abs(emp - ps.probabilities(st)).sum() < 0.005

    def test_zero_probability_never_drawn(self):
        st = ps.new_state(3)
        st.amps[:] = 0
        st.amps[[2, 5]] = R2
        assert set(ps.sample(st, 10_000, seed=8).counts) == {2, 5}

    def test_sample_count_validated(self):
        with pytest.raises(ValueError):
            ps.sample(ps.new_state(1), 0)

    def test_all_zero_rejected(self):
        dead = ps.StateVector(2, np.zeros(4, dtype=np.complex64))
        with pytest.raises(ps.DegenerateStateError):
            ps.sample(dead, 10)
        with pytest.raises(ps.DegenerateStateError):
            ps.measure_collapse(dead, seed=0)

    def test_collapse_one_hot_phase_discarded(self):
        for seed in range(50):
            st = ps.new_state(1)
            st.amps[:] = [0.6, 0.8j]
            m, after = ps.measure_collapse(st, seed=seed)
            if m == 1:
                assert after.amps[1] == 1.0 + 0.0j
                break
        else:
            pytest.fail("outcome 1 never drawn")

    def test_histogram_formats(self):
        h = ps.MeasurementHistogram({3: 10, 0: 5}, 15)
        assert h.to_csv() == "basis_index,count\n0,5\n3,10\n"
        assert ps.MeasurementHistogram.from_outcomes(np.array([1, 1, 2, 1])).counts == {1: 3, 2: 1}


class TestState:  # pkg/tests/test_state.py
    def test_one_hot(self):
        np.testing.assert_array_equal(ps.new_state(3).amps, [1, 0, 0, 0, 0, 0, 0, 0])

    def test_accessor(self):
        st = ps.new_state(4)
        assert [ps.amplitude_of(st, j) for j in range(16)] == [1] + [0] * 15

    def test_capacity_message(self):
        with pytest.raises(ps.CapacityError) as e:
            ps.new_state(30, memory_budget=8_000_000_000)
        assert "8589934592" in str(e.value)

    def test_memory_table(self):
        for n, text in [(5, "256 B"), (10, "8.192 kB"), (20, "8.389 MB"), (25, "268.4 MB"), (30, "8.59 GB")]:
            assert ps.format_bytes(ps.memory_required(n) // 8) == text

    def test_double_register(self):
        """Precision.DOUBLE lives on the device as complex128 (state.py:25-42);
        its budget check counts 16 bytes per amplitude (state.py:71-83)."""
        sv = ps.new_state(2, ps.Precision.DOUBLE)
        assert sv.precision is ps.Precision.DOUBLE
        assert sv.amps.dtype == np.complex128 and sv.amps[0] == 1
        with pytest.raises(ps.CapacityError):
            ps.new_state(10, ps.Precision.DOUBLE, memory_budget=16 * 1024 - 1)
        ps.new_state(10, ps.Precision.DOUBLE, memory_budget=16 * 1024)

    def test_amplitude_out_of_range(self):
        with pytest.raises(IndexError):
            ps.amplitude_of(ps.new_state(2), 4)


class TestCircuits:  # pkg/tests/test_circuits.py
    def test_bell(self):
        st, _ = ps.run_circuit(ps.Circuit(2, (ps.Apply(ps.H, 0), ps.ControlledApply(ps.X, 0, 1))))
        np.testing.assert_allclose(st.amps, [R2, 0, 0, R2], atol=1e-7)

    def test_histogram_filled(self):
        _, h = ps.run_circuit(ps.Circuit(2, (ps.Apply(ps.X, 1), ps.SampleMeasure(50))), seed=4)
        assert h.counts == {2: 50}

    def test_qft_uniform(self):
        st, _ = ps.run_circuit(ps.build_qft(4))
        np.testing.assert_allclose(st.amps, np.full(16, 0.25), atol=1e-6)

    @pytest.mark.parametrize("n", range(1, 7))
    def test_qft_dft_bit_reversal(self, n):
        dim = 1 << n
        omega = np.exp(2j * np.pi / dim)
        dft = omega ** np.outer(np.arange(dim), np.arange(dim)) / np.sqrt(dim)
        for x in range(dim):
            st = ps.new_state(n)
            st.amps[:] = 0
            st.amps[x] = 1
            for ins in ps.build_qft(n).instructions:
                if isinstance(ins, ps.Apply):
                    ps.apply_gate(st, ins.target, ins.gate)
                else:
                    ps.apply_controlled_gate(st, ins.control, ins.target, ins.gate)
            rev = int(format(x, f"0{n}b")[::-1], 2)
            np.testing.assert_allclose(st.amps, dft[:, rev], atol=1e-5)

    def test_bernstein_vazirani(self):
        _, h = ps.run_circuit(ps.build_bernstein_vazirani(14, 101, shots=1000), seed=20260808)
        assert h.counts == {101: 1000}
        for hidden in range(0, 256, 17):
            _, h = ps.run_circuit(ps.build_bernstein_vazirani(8, hidden, shots=16), seed=hidden)
            assert h.counts == {hidden: 16}

    def test_normalization_drift_10k(self):  # pkg/tests/test_acceptance.py:149-162
        rng = np.random.default_rng(99)
        st = ps.new_state(10)
        gates = [ps.random_unitary_gate(rng) for _ in range(64)]
        dev = st.device_state
        for _ in range(10_000):
            t = int(rng.integers(10))
            g = gates[int(rng.integers(len(gates)))]
            if rng.random() < 0.3:
                c = int(rng.integers(9))
                dev.apply_controlled_gate(g, c + (c >= t), t)
            else:
                dev.apply_gate(g, t)
        assert abs(ps.norm_squared(st) - 1.0) < 1e-3


class TestMirrorTracking:
    """A handed-out `amps` is re-uploaded only after the host wrote to it."""

    def test_reads_do_not_force_uploads(self):
        st = ps.new_state(8)
        ps.apply_gate(st, 0, ps.H)
        a = st.amps  # handed out
        for t in range(1, 8):
            ps.apply_gate(st, t, ps.H)
        assert st._uploads == 0 and a is st.amps
        assert np.allclose(a, np.full(256, 1 / 16, np.complex64), atol=1e-6)
        _ = float(np.abs(a).sum()), a.tobytes(), a.copy()
        ps.apply_gate(st, 3, ps.H)
        assert st._uploads == 0

    @pytest.mark.parametrize("write", ["setitem", "slice_view", "inplace", "copyto", "fill", "real"])
    def test_every_write_path_reaches_the_device(self, write):
        st = ps.new_state(5)
        a = st.amps
        if write == "setitem":
            a[3] = 1
        elif write == "slice_view":
            v = a[2:6]
            v[1] = 1
        elif write == "inplace":
            a += np.eye(1, 32, 3, dtype=np.complex64)[0]
        elif write == "copyto":
            np.copyto(a, np.eye(1, 32, 3, dtype=np.complex64)[0])
        elif write == "fill":
            a.fill(0)
            a[3] = 1
        else:
            a.real[3] = 1
        if write != "copyto" and write != "fill":
            a[0] = 0
        ps.apply_gate(st, 1, ps.X)
        assert st._uploads == 1
        expect = np.zeros(32, np.complex64)
        expect[3 ^ 2] = 1
        np.testing.assert_array_equal(st.amps, expect)
