"""The single-process multi-device C ABI (qs_create_sharded, csrc/sharded.cu)
through MultiDeviceState.  On the one-GPU box the shards repeat device 0,
which exercises the same host logic (qubit map, swaps, predicates,
canonicalisation, the chained CDF) with the peer-memory exchange; results
must equal the unsharded register bit for bit."""

from __future__ import annotations

import numpy as np
import pytest

from golden_util import same_values
from paper_1805_00988_b200 import Circuit, State, build_hadamard_layer, build_qft, execute, u1
from paper_1805_00988_b200.circuits import Apply, ControlledApply
from paper_1805_00988_b200.gates import FIXED_GATES
from paper_1805_00988_b200.multigpu import MultiDeviceState
from test_sharded import mixed_circuit

pytestmark = pytest.mark.gpu


def _circ(n, seed):
    ins = build_hadamard_layer(n).instructions + mixed_circuit(n, 150, seed).instructions
    # diagonal gates whose bits are all global (whole-shard multiplies)
    ins += (ControlledApply(u1(0.37), n - 1, n - 2), Apply(FIXED_GATES["t"], n - 1))
    return Circuit(n, ins + build_qft(n).instructions[-50:])


@pytest.mark.parametrize("n,shards,peer_gates", [(12, 2, False), (14, 4, False), (14, 4, True), (16, 8, True),
                                                  (20, 4, False)])
def test_equals_unsharded(n, shards, peer_gates):
    circ = _circ(n, 7 * n + shards)
    ref = State(n)
    execute(circ, ref, fuse=False)
    with MultiDeviceState(n, [0] * shards, peer_gates=peer_gates) as reg:
        reg.run(circ)
        st = reg.stats()
        assert st["exchange"] == "p2p"
        assert (st["peer_gates"] > 0) if peer_gates else (st["swaps"] > 0)
        assert same_values(reg.amplitudes(), ref.amplitudes())
        assert reg.probabilities().tobytes() == ref.probabilities().tobytes()
        assert np.array_equal(reg.sample_outcomes(5000, 11), ref.sample_outcomes(5000, 11))
        assert abs(reg.norm_squared() - ref.norm_squared()) < 1e-9
        # partial reads across a shard boundary
        L = reg.shard_qubits
        lo = (1 << L) - 5
        assert same_values(reg.amplitudes(lo, 10), ref.amplitudes(lo, 10))
    ref.close()


def test_set_amplitudes_reset_and_errors():
    n = 13
    rng = np.random.default_rng(3)
    v = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)).astype(np.complex64)
    with MultiDeviceState(n, [0, 0, 0, 0]) as reg:
        reg.set_amplitudes(v)
        assert same_values(reg.amplitudes(), v)
        reg.h(n - 1)  # global target: one swap
        ref = State(n)
        ref.set_amplitudes(v)
        ref.h(n - 1)
        assert same_values(reg.amplitudes(), ref.amplitudes())
        reg.reset(5 | (1 << (n - 1)))
        a = reg.amplitudes()
        assert a[5 | (1 << (n - 1))] == 1 and np.count_nonzero(a) == 1
        with pytest.raises(IndexError):
            reg.h(n)
        with pytest.raises(ValueError):
            reg.cx(3, 3)
        reg.reset(0)
        reg.set_amplitudes(np.zeros(1 << n, np.complex64))
        from paper_1805_00988_b200 import DegenerateStateError

        with pytest.raises(DegenerateStateError):
            reg.sample_outcomes(10, 1)
    with pytest.raises(ValueError):
        MultiDeviceState(10, [0, 0, 0])
    with pytest.raises(IndexError):
        MultiDeviceState(10, [0, 99])


def test_generator_seed_advances():
    n = 12
    with MultiDeviceState(n, [0, 0]) as reg:
        reg.run(build_hadamard_layer(n))
        g1, g2 = np.random.default_rng(5), np.random.default_rng(5)
        a = reg.sample_outcomes(100, g1)
        b = reg.sample_outcomes(100, g1)
        ref = State(n)
        execute(build_hadamard_layer(n), ref, fuse=False)
        assert np.array_equal(a, ref.sample_outcomes(100, g2)) and np.array_equal(b, ref.sample_outcomes(100, g2))
        assert not np.array_equal(a, b)
        ref.close()


def test_fused_passes_on_two_devices_in_one_process():
    """kernel attributes are per device; a fused pass on device 1
    after device 0 must launch (needs 2 GPUs; skipped on the one-GPU box)."""
    from paper_1805_00988_b200 import _native as N

    if N.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    n = 20
    outs = []
    for dev in (0, 1):
        st = State(n, device=dev)
        execute(build_qft(n), st, fuse=True)
        outs.append(st.amplitudes())
        st.close()
    assert same_values(outs[0], outs[1])


@pytest.mark.parametrize("n,shards,peer_gates", [(14, 4, False), (16, 2, True), (22, 4, False)])
def test_fused_run_equals_unsharded(n, shards, peer_gates):
    """MultiDeviceState.run with fused local passes on the shards between the
    C ABI's global gates == the unsharded register, bitwise."""
    circ = _circ(n, 3 * n + shards)
    ref = State(n)
    execute(circ, ref, fuse=False)
    with MultiDeviceState(n, [0] * shards, peer_gates=peer_gates) as reg:
        reg.run(circ, fuse=True)
        assert same_values(reg.amplitudes(), ref.amplitudes())
        assert np.array_equal(reg.sample_outcomes(2000, 3), ref.sample_outcomes(2000, 3))
    ref.close()


def test_fused_run_inexact_to_tolerance():
    from paper_1805_00988_b200 import fusion

    n = 20
    circ = Circuit(n, build_hadamard_layer(n).instructions + build_qft(n).instructions)
    ref = State(n)
    execute(circ, ref, fuse=False)
    with MultiDeviceState(n, [0, 0, 0, 0]) as reg:
        reg.run(circ, exact=False)
        fusion.jit_sync()
        reg.reset(0)
        reg.run(circ, exact=False)
        np.testing.assert_allclose(reg.amplitudes(), ref.amplitudes(), rtol=1e-5, atol=1e-5 * 2.0 ** (-n / 2))
    ref.close()
