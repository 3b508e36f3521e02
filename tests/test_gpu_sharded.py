"""Sharded registers on the GPU: P virtual shards on one B200 run the same
ShardedState swap logic as the multi-process NCCL path; results must equal the
unsharded register bit for bit (values)."""

from __future__ import annotations

import numpy as np
import pytest

from golden_util import same_values
from paper_1805_00988_b200 import Circuit, State, build_hadamard_layer, build_qft, execute
from paper_1805_00988_b200.sharded import ShardedState
from test_sharded import mixed_circuit

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,shards", [(12, 2), (14, 4), (16, 8), (22, 4)])
def test_virtual_shards_equal_unsharded(n, shards):
    circ = Circuit(n, build_hadamard_layer(n).instructions + mixed_circuit(n, 80, n).instructions
                   + build_qft(n).instructions)
    ref = State(n)
    execute(circ, ref, fuse=False)
    st = ShardedState.virtual(n, shards)
    st.run(circ)
    assert st.swaps > 0
    assert same_values(st.amplitudes(), ref.amplitudes())
    assert st.probabilities().tobytes() == ref.probabilities().tobytes()


def test_gate_api_and_canonicalize_roundtrip():
    n = 13
    st = ShardedState.virtual(n, 4)
    ref = State(n)
    for q in range(n):
        st.h(q)
        ref.h(q)
    st.cx(n - 1, 0)
    ref.cx(n - 1, 0)
    st.ccx(n - 2, n - 1, 3)
    ref.ccx(n - 2, n - 1, 3)
    st.cu1(n - 1, n - 2, 0.7)
    ref.cu1(n - 1, n - 2, 0.7)
    assert same_values(st.amplitudes(), ref.amplitudes())
    assert st.layout.is_identity()


@pytest.mark.parametrize("n,shards", [(12, 2), (16, 4), (20, 8)])
def test_sharded_sampling_equals_unsharded(n, shards):
    circ = Circuit(n, mixed_circuit(n, 60, 3 * n).instructions)
    ref = State(n)
    execute(circ, ref, fuse=False)
    st = ShardedState.virtual(n, shards)
    st.run(circ)
    for seed in (1, 77):
        assert np.array_equal(st.sample_outcomes(5000, seed), ref.sample_outcomes(5000, seed))
    assert st.measure(1000, seed=4) == ref.measure(1000, seed=4)


@pytest.mark.parametrize("n,shards", [(12, 2), (16, 4), (20, 8)])
def test_peer_gates_equal_unsharded(n, shards):
    """Global-target gates through csrc/peer.cu (partner shards on the same GPU
    stand in for NVLink peers): no swaps, same bits as the unsharded register."""
    circ = Circuit(n, build_hadamard_layer(n).instructions + mixed_circuit(n, 80, n + 1).instructions
                   + build_qft(n).instructions)
    ref = State(n)
    execute(circ, ref, fuse=False)
    st = ShardedState.virtual(n, shards, peer_gates=True)
    st.run(circ)
    assert st.peer_gate_count > 0
    assert same_values(st.amplitudes(), ref.amplitudes())


def test_auto_global_gate_mode_equals_unsharded():
    n = 16
    circ = Circuit(n, build_hadamard_layer(n).instructions + mixed_circuit(n, 100, 5).instructions)
    ref = State(n)
    execute(circ, ref, fuse=False)
    st = ShardedState.virtual(n, 4, peer_gates="auto")
    st.run(circ)
    assert st.calibration is not None
    assert same_values(st.amplitudes(), ref.amplitudes())
    st.close()


def test_inexact_sharded_run_to_tolerance():
    from paper_1805_00988_b200 import fusion

    n = 18
    circ = Circuit(n, build_hadamard_layer(n).instructions + build_qft(n).instructions)
    ref = State(n)
    execute(circ, ref, fuse=False)
    st = ShardedState.virtual(n, 4)
    st.run(circ, exact=False)
    fusion.jit_sync()
    st.reset(0)
    st.run(circ, exact=False)
    np.testing.assert_allclose(st.amplitudes(), ref.amplitudes(), rtol=1e-5, atol=1e-5 * 2.0 ** (-n / 2))
    st.close()


@pytest.mark.parametrize("peer_gates,exchange", [(False, "nccl"), (False, "peer"), (True, "peer")])
def test_complex128_shards_equal_unsharded(peer_gates, exchange):
    """Precision.DOUBLE registers sharded: swaps (copies or the peer swap
    kernel) and peer gates on 16-B amplitudes, bit-exact vs the unsharded
    complex128 register, probabilities and draws included."""
    n = 14
    circ = Circuit(n, build_hadamard_layer(n).instructions + mixed_circuit(n, 90, 21).instructions
                   + build_qft(n).instructions[-30:])
    ref = State(n, precision="double")
    execute(circ, ref, fuse=False)
    st = ShardedState.virtual(n, 4, peer_gates=peer_gates, exchange=exchange, precision="double")
    st.run(circ)
    a = st.amplitudes()
    assert a.dtype == np.complex128 and same_values(a, ref.amplitudes())
    assert st.probabilities().tobytes() == ref.probabilities().tobytes()
    assert np.array_equal(st.sample_outcomes(3000, 5), ref.sample_outcomes(3000, 5))
    st.close()
    ref.close()
