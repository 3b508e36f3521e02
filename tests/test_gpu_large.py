"""GPU parity past 2^31 amplitudes (BASELINE config 4 at n = 32; SURVEY 8(d)
row 4 "fused == unfused bitwise on the GPU at n = 32").

Indices above 2^31 are where 32-bit index arithmetic would break, so besides
whole-register properties these tests check exact values at HIGH addresses:
two 2^20-amplitude blocks B0 (bit 31 = 0) and B1 = B0 + 2^31 are loaded with
random amplitudes; every op of the circuit pairs bits inside {0..19, 31} (or
is controlled by bits 20..30, whose value the blocks fix), so the blocks
evolve as a closed 21-qubit register — which the oracle computes.

Whole-register comparisons run on the device (zero-copy torch views of the
registers, chunked), so 32 GiB registers need no host round trip.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from golden_util import M8Gate, same_values
from oracle import c as oc
from paper_1805_00988_b200 import (
    FIXED_GATES,
    State,
    build_hadamard_layer,
    build_qft,
    execute,
    layered_random_circuit,
    random_unitary_gate,
    u1,
)
from paper_1805_00988_b200.circuits import Apply, Circuit, ControlledApply, ControlledControlledApply

pytestmark = pytest.mark.gpu

H, T, X = FIXED_GATES["h"], FIXED_GATES["t"], FIXED_GATES["x"]


def view(st: State) -> torch.Tensor:
    """float32 (2 * 2^n,) device view of a register (no copy)."""
    ptr = st.device_pointer()
    nfloat = 2 << st.num_qubits

    class _CAI:
        __cuda_array_interface__ = {"shape": (nfloat,), "typestr": "<f4", "data": (ptr, False),
                                    "version": 3, "strides": None}

    st.flush()
    return torch.as_tensor(_CAI(), device=torch.device("cuda", st.device))


def device_equal(a: torch.Tensor, b: torch.Tensor, chunk: int = 1 << 28) -> bool:
    """Value equality (+0 == -0, the sign-of-zero freedom DESIGN.md documents)."""
    assert a.numel() == b.numel()
    for off in range(0, a.numel(), chunk):
        if not torch.equal(a[off: off + chunk], b[off: off + chunk]):
            return False
    return True


def load(n: int, amps) -> State:
    st = State(n)
    st.set_amplitudes(amps)
    return st


def free_gib() -> float:
    return torch.cuda.mem_get_info()[0] / 2**30


def need(gib: float):
    if free_gib() < gib:
        pytest.skip(f"needs {gib} GiB of free HBM")


class TestConfig4At32:
    def test_layered_random_fused_equals_unfused(self):
        """config 4 exactly as benchmarked: layered_random_circuit(32, 20, seed=32),
        fused passes (TMA tiles) vs one sweep per gate, all 2^32 amplitudes."""
        need(66)
        n = 32
        circ = layered_random_circuit(n, 20, seed=32)
        fused, plain = State(n), State(n)
        execute(circ, fused, fuse=True)
        execute(circ, plain, fuse=False)
        assert device_equal(view(fused), view(plain))
        assert abs(fused.norm_squared() - 1.0) < 1e-3
        fused.close()
        plain.close()

    def test_generator_matches_smaller_widths(self):
        """The same generator at n = 22 vs the oracle (bit-exact, unfused and fused)."""
        n = 22
        circ = layered_random_circuit(n, 20, seed=32)
        ref = np.zeros(1 << n, np.complex64)
        ref[0] = 1
        for ins in circ.instructions:
            if isinstance(ins, Apply):
                oc.apply_gate(ref, ins.target, ins.gate)
            else:
                oc.apply_controlled_gate(ref, ins.control, ins.target, ins.gate)
        for fuse in (False, True):
            st = State(n)
            execute(circ, st, fuse=fuse)
            assert same_values(st.amplitudes(), ref), fuse
            st.close()


class TestWholeRegister32:
    def test_hlayer32_uniform(self):
        """H on all 32 qubits from |0>: every amplitude is the sequentially
        rounded (1/sqrt2)^32, imaginary parts zero, fused and unfused."""
        need(34)
        n = 32
        v = np.float32(1.0)
        h = np.float32(1 / math.sqrt(2))
        for _ in range(n):
            v = np.float32(h * v)
        for fuse in (False, True):
            st = State(n)
            execute(build_hadamard_layer(n), st, fuse=fuse)
            w = view(st).view(-1, 2)
            chunk = 1 << 27
            for off in range(0, w.shape[0], chunk):
                c = w[off: off + chunk]
                assert bool((c[:, 0] == float(v)).all()) and bool((c[:, 1] == 0).all()), (fuse, off)
            st.close()

    def test_round_trip_every_target_n32(self):
        """U then U^dagger on every target of a 32-qubit entangled register."""
        need(66)
        n = 32
        rng = np.random.default_rng(32)
        st = State(n)
        execute(build_hadamard_layer(n), st, fuse=True)
        for q in range(0, n, 3):
            st.t(q)
        st.cx(31, 0)
        st.cx(2, 30)
        before = State(n)
        torch_before = view(before)
        torch_before.copy_(view(st))
        torch.cuda.synchronize()  # the copy runs on torch's stream, the gates on the register's
        g = random_unitary_gate(rng)
        for t in range(n):
            st.apply_gate(g, t)
            st.apply_gate(g.dagger(), t)
        a, b = view(st), torch_before
        chunk = 1 << 28
        worst = 0.0
        for off in range(0, a.numel(), chunk):
            worst = max(worst, float((a[off: off + chunk] - b[off: off + chunk]).abs().max()))
        assert worst < 1e-5 * 2.0 ** (-n / 2) * 16
        assert abs(st.norm_squared() - 1.0) < 1e-3
        st.close()
        before.close()


# ---- exact values at high addresses --------------------------------------------
OFF = (1 << 30) | (1 << 29) | (1 << 25) | (1 << 23) | (1 << 20)  # bits 20..30 fixed by the blocks; bit 31 = 0
BLK = 1 << 20
HIGH = 31


def _sub_op(ins):
    """The op as seen by the 21-qubit sub-register (global 31 -> sub 20), or
    None when a control on bits 20..30 is 0 on the blocks."""
    def sub(q):
        return 20 if q == HIGH else q

    if isinstance(ins, Apply):
        return ("g", sub(ins.target), [], ins.gate)
    ctrls = [ins.control] if isinstance(ins, ControlledApply) else [ins.control1, ins.control2]
    keep = []
    for c in ctrls:
        if 20 <= c <= 30:
            if not (OFF >> c) & 1:
                return None
        else:
            keep.append(sub(c))
    return ("g", sub(ins.target), keep, ins.gate)


def _oracle_apply(ref, op):
    _, t, ctrls, gate = op
    if not ctrls:
        oc.apply_gate(ref, t, gate)
    elif len(ctrls) == 1:
        oc.apply_controlled_gate(ref, ctrls[0], t, gate)
    else:
        oc.apply_cc_gate(ref, ctrls[0], ctrls[1], t, gate)


def high_circuit(rng):
    """Gates on targets in {0..19, 31} with controls anywhere (bits 20..30 act
    as fixed predicates on the blocks)."""
    g1, g2 = random_unitary_gate(rng), random_unitary_gate(rng)
    tg = [0, 1, 5, 6, 7, 12, 19, HIGH]
    ins = [Apply(H, HIGH), Apply(g1, 0), Apply(g2, HIGH), Apply(g1, 6), Apply(g2, 19)]
    ins += [ControlledApply(X, HIGH, 3), ControlledApply(g1, 4, HIGH), ControlledApply(u1(0.7), HIGH, 9)]
    ins += [ControlledApply(g2, 29, HIGH), ControlledApply(g2, 21, 5),  # bit 29 set in OFF, bit 21 clear (skipped)
            ControlledApply(u1(1.1), 28, HIGH),  # bit 28 clear: skipped
            ControlledControlledApply(X, HIGH, 2, 11),
            ControlledControlledApply(g1, 25, 3, HIGH)]  # bit 25 set
    for _ in range(40):
        t = int(rng.choice(tg))
        c = int(rng.choice([q for q in list(range(20)) + [HIGH] if q != t]))
        ins.append(ControlledApply(u1(float(rng.random())), c, t) if rng.random() < 0.4 else Apply(g1 if rng.random() < 0.5 else g2, t))
    return Circuit(32, tuple(ins))


class TestHighAddresses:
    @pytest.mark.parametrize("fuse", [False, True])
    def test_blocks_above_2_31(self, fuse):
        assert (OFF >> 29) & 1 and (OFF >> 25) & 1 and not (OFF >> 21) & 1 and not (OFF >> 28) & 1
        assert not (OFF >> 31) & 1 and OFF % BLK == 0
        need(34)
        rng = np.random.default_rng(2031)
        n = 32
        b0 = (rng.normal(size=BLK) + 1j * rng.normal(size=BLK)).astype(np.complex64) * np.float32(1e-3)
        b1 = (rng.normal(size=BLK) + 1j * rng.normal(size=BLK)).astype(np.complex64) * np.float32(1e-3)
        st = State(n)
        st.set_amplitudes(b0, offset=OFF)
        st.set_amplitudes(b1, offset=OFF + (1 << HIGH))
        circ = high_circuit(rng)
        execute(circ, st, fuse=fuse)
        ref = np.concatenate([b0, b1])
        for ins in circ.instructions:
            op = _sub_op(ins)
            if op is not None:
                _oracle_apply(ref, op)
        got0 = st.amplitudes(OFF, BLK)
        got1 = st.amplitudes(OFF + (1 << HIGH), BLK)
        assert same_values(got0, ref[:BLK])
        assert same_values(got1, ref[BLK:])
        st.close()

    def test_basis_state_above_2_31(self):
        need(34)
        n = 32
        x = (1 << 31) | (1 << 30) | 0x12345
        st = State(n).reset(x)
        st.x(31)
        st.cx(30, 0)
        assert st.amplitude(x ^ (1 << 31) ^ 1) == 1
        st.ccx(30, 16, 31)  # bit 16 of x is set: flips bit 31 back
        assert st.amplitude(x ^ 1) == 1
        execute(build_qft(n), st, fuse=True)
        # QFT|x'>[k] = exp(2 pi i k rev(x') / N) / sqrt(N), x' = x ^ 1
        rev = int(format(x ^ 1, f"0{n}b")[::-1], 2)
        ks = np.array([0, 1, (1 << 31) + 5, (1 << 32) - 1, 0x9ABCDEF1, 0x7FFFFFFF, 0x80000000], dtype=np.int64)
        got = np.array([st.amplitude(int(k)) for k in ks])
        want = np.exp(2j * np.pi * ((ks * rev) % (1 << n)) / (1 << n)) / math.sqrt(1 << n)
        assert np.max(np.abs(got - want)) < 1e-3 * abs(want[0])
        st.close()


    def test_from_basis_above_2_31(self):
        """execute(..., initial_basis=x) on a 32-qubit register holding other
        data: the first fused pass writes |x>'s tiles (x above 2^31); equal to
        reset(x) + the same passes over all 2^32 amplitudes."""
        need(70)
        n = 32
        x = (1 << 31) | (1 << 29) | 0x2345
        circ = Circuit(n, build_qft(n).instructions[:200])
        states = []
        for folded in (False, True):
            st = State(n)
            for q in range(0, n, 3):
                st.h(q)  # stale contents the folded reset must overwrite
            if folded:
                execute(circ, st, fuse=True, initial_basis=x)
            else:
                st.reset(x)
                execute(circ, st, fuse=True)
            states.append(st)
        assert device_equal(view(states[0]), view(states[1]))
        for st in states:
            st.close()


class TestShardedAt31:
    def test_two_virtual_shards_equal_unsharded(self):
        """A 31-qubit register as two 30-qubit shards (qubit 30 global: qubit
        swaps through the exchange) == the unsharded register, bitwise."""
        need(40)
        from paper_1805_00988_b200.sharded import ShardedState

        n = 31
        rng = np.random.default_rng(31)
        g = random_unitary_gate(rng)
        ins = [Apply(H, q) for q in range(n)]
        ins += [Apply(T, 30), ControlledApply(X, 30, 3), ControlledApply(g, 2, 30), Apply(g, 30),
                ControlledApply(u1(0.3), 30, 29), ControlledControlledApply(X, 30, 1, 17), Apply(H, 29)]
        ins += list(build_qft(n).instructions[-40:])
        circ = Circuit(n, tuple(ins))
        ref = State(n)
        execute(circ, ref, fuse=False)
        for peer in (False, True):
            sh = ShardedState.virtual(n, 2, peer_gates=peer)
            sh.run(circ)
            sh.canonicalize()
            rv = view(ref)
            half = rv.numel() // 2
            for r, eng in zip(sh.ranks, sh.engines):
                eng.synchronize()
                assert device_equal(eng.view(), rv[r * half:(r + 1) * half]), (peer, r)
            sh.close()
        ref.close()


class TestReorderedPlanner:
    """The opt-in commutation-aware planner (fusion.plan(reorder=True)):
    agreement with the reference to the north_star tolerance."""

    @pytest.mark.parametrize("n", [20, 24])
    def test_layered_to_tolerance(self, n):
        circ = layered_random_circuit(n, 20, seed=32)
        a, b = State(n), State(n)
        execute(circ, a, fuse=True, reorder=True)
        execute(circ, b, fuse=False)
        x, y = a.amplitudes(), b.amplitudes()
        np.testing.assert_allclose(x, y, rtol=1e-5, atol=1e-5 * 2.0 ** (-n / 2))
        a.close()
        b.close()

    def test_config4_n32_to_tolerance(self):
        need(66)
        n = 32
        circ = layered_random_circuit(n, 20, seed=32)
        a, b = State(n), State(n)
        execute(circ, a, fuse=True, reorder=True)
        execute(circ, b, fuse=True)
        va, vb = view(a), view(b)
        chunk = 1 << 28
        worst = 0.0
        for off in range(0, va.numel(), chunk):
            worst = max(worst, float((va[off: off + chunk] - vb[off: off + chunk]).abs().max()))
        assert worst <= 1e-5 * 2.0 ** (-n / 2) * 4
        a.close()
        b.close()


class TestInexactMode:
    """execute(..., exact=False): commutation-aware passes + combined diagonal
    runs (QS_FUSED_COMBINE_PHASES) — equal to the reference to the north_star
    tolerance (rtol 1e-5), not bit for bit.  Compiled programs only, so the
    compiles are waited for before the timed/compared run."""

    @pytest.mark.parametrize("n,name", [(20, "qft"), (24, "qft"), (22, "layered"), (21, "random")])
    def test_matches_exact_to_tolerance(self, n, name):
        from paper_1805_00988_b200 import fusion, random_circuit

        circ = {"qft": lambda: build_qft(n), "layered": lambda: layered_random_circuit(n, 12, seed=3),
                "random": lambda: random_circuit(n, 300, np.random.default_rng(5))}[name]()
        a, b = State(n), State(n)
        rng = np.random.default_rng(n)
        v = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)).astype(np.complex64)
        v /= np.float32(np.linalg.norm(v))
        a.set_amplitudes(v)
        execute(circ, a, fuse=True, exact=False)
        fusion.jit_sync()
        a.set_amplitudes(v)
        execute(circ, a, fuse=True, exact=False)
        b.set_amplitudes(v)
        execute(circ, b, fuse=False)
        np.testing.assert_allclose(a.amplitudes(), b.amplitudes(), rtol=1e-5, atol=1e-5 * 2.0 ** (-n / 2))
        a.close()
        b.close()

    def test_qft30_analytic(self):
        """QFT|x> (no swaps) = exp(2 pi i k rev(x) / N) / sqrt(N) at n = 30."""
        from paper_1805_00988_b200 import fusion

        n = 30
        x = 0b101100111000111100001011010110
        st = State(n).reset(x)
        execute(build_qft(n), st, fuse=True, exact=False)
        fusion.jit_sync()
        st.reset(x)
        execute(build_qft(n), st, fuse=True, exact=False)
        rev = int(format(x, f"0{n}b")[::-1], 2)
        ks = np.arange(0, 1 << n, 1 << 17, dtype=np.int64)[:300] + 12345
        got = np.array([st.amplitude(int(k)) for k in ks])
        want = np.exp(2j * np.pi * ((ks * rev) % (1 << n)) / (1 << n)) / math.sqrt(1 << n)
        np.testing.assert_allclose(got, want, rtol=1e-4, atol=1e-4 * abs(want[0]))
        st.close()


class TestReadout:
    def test_probabilities_into_pinned_array(self):
        """State.probabilities(out=pinned_empty(...)): the DMA path gives the
        bytes of the staged path (and of the oracle)."""
        from paper_1805_00988_b200 import _native as N

        n = 21
        rng = np.random.default_rng(21)
        v = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)).astype(np.complex64)
        st = State(n)
        st.set_amplitudes(v)
        fresh = st.probabilities()
        pin = N.pinned_empty(1 << n)
        got = st.probabilities(out=pin)
        assert got is pin and got.tobytes() == fresh.tobytes() == oc.probabilities(v).tobytes()
        part = N.pinned_empty(1000)
        assert st.probabilities(12345, 1000, out=part).tobytes() == fresh[12345:13345].tobytes()
        with pytest.raises(ValueError):
            st.probabilities(out=np.empty(10))
        st.close()


class TestCheckpoint:
    @pytest.mark.parametrize("precision", ["single", "double"])
    def test_save_load_round_trip(self, tmp_path, precision):
        from paper_1805_00988_b200 import fusion

        n = 18
        st = State(n, precision=precision)
        execute(build_qft(n), st, fuse=False)
        st.t(3)
        st.cx(17, 2)
        path = tmp_path / "reg.npy"
        st.save(path)
        back = State.load(path)
        assert back.num_qubits == n and back.dtype == st.dtype
        assert back.amplitudes().tobytes() == st.amplitudes().tobytes()
        assert np.load(path).tobytes() == st.amplitudes().tobytes()
        st.close()
        back.close()


class TestSamplingChainPaths:
    """Per-draw parity of the exact sampling chain on states that force each
    of its paths at 2^22 amplitudes (4 blocks of 256 chunks): binade
    crossings inside chunks and sub-blocks (log-uniform magnitudes), an
    all-zero prefix (all-exact0 blocks), a basis state (exact0 chunk with
    absolute fine starts), a uniform state (30 crossings)."""

    @pytest.mark.parametrize("kind", ["loguniform", "zero_prefix", "basis", "uniform", "spiky", "scaled_up",
                                      "scaled_down"])
    def test_per_draw_vs_oracle(self, kind):
        n = 22
        rng = np.random.default_rng(hash(kind) % 1000)
        if kind == "loguniform":
            mag = np.exp(rng.uniform(np.log(1e-30), 0.0, size=1 << n))
            amps = (mag * np.exp(2j * np.pi * rng.random(1 << n))).astype(np.complex64)
        elif kind == "zero_prefix":
            amps = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)).astype(np.complex64)
            amps[: (3 << n) // 4] = 0
        elif kind == "basis":
            amps = np.zeros(1 << n, np.complex64)
            amps[3_000_001] = 1
        elif kind == "uniform":
            amps = np.full(1 << n, np.float32(2.0 ** (-n / 2)), np.complex64)
        elif kind in ("scaled_up", "scaled_down"):  # unnormalised: total 2^22 * 1e12 or * 1e-34
            scale = 1e6 if kind == "scaled_up" else 1e-17
            amps = ((rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)) * scale).astype(np.complex64)
        else:  # a few large spikes on a tiny floor
            amps = np.full(1 << n, np.float32(1e-20), np.complex64)
            amps[rng.integers(0, 1 << n, 40)] = rng.normal(size=40).astype(np.float32)
        st = load(n, amps)
        for seed in (1, 77):
            got = st.sample_outcomes(20000, seed)
            assert np.array_equal(got, oc.sample_outcomes(amps, 20000, seed)), (kind, seed)
        st.close()


@pytest.mark.parametrize("n", [16, 17, 18, 19])
def test_sampling_m3_forms_at_the_warp_boundary(n):
    """M3 runs register-staged below 32 chunks (n < 17) and as the bulk-copy
    ring from whole warps of chunks on (n >= 17): per-draw parity with the
    oracle on both sides of the boundary, on a state with binade crossings
    inside chunks (log-uniform magnitudes) and on a uniform one."""
    rng = np.random.default_rng(n)
    mag = np.exp(rng.uniform(np.log(1e-20), 0.0, size=1 << n))
    for amps in ((mag * np.exp(2j * np.pi * rng.random(1 << n))).astype(np.complex64),
                 np.full(1 << n, np.float32(2.0 ** (-n / 2)), np.complex64)):
        st = load(n, amps)
        got = st.sample_outcomes(5000, 9)
        assert np.array_equal(got, oc.sample_outcomes(amps, 5000, 9))
        st.close()
