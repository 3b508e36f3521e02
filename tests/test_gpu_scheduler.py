"""The fused passes' dynamic tile scheduler (csrc/fused_dev.cuh: one atomic
counter per handle, zeroed by the last CTA of every launch): passes on
several handles interleaved on their own streams, handles recycled through
the buffer cache, and passes whose tiles differ in work (tile-uniform tests)
all give the bits of the per-op sweeps."""

from __future__ import annotations

import os

import numpy as np
import pytest

from golden_util import same_values
from paper_1805_00988_b200 import State, build_qft, execute, fusion, layered_random_circuit, u1
from paper_1805_00988_b200.circuits import Apply, Circuit, ControlledApply, lower_ops

pytestmark = pytest.mark.gpu


def rand_amps(n, seed):
    rng = np.random.default_rng(seed)
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return (v / np.linalg.norm(v)).astype(np.complex64)


def reference(circ, a0):
    st = State(circ.num_qubits)
    st.set_amplitudes(a0)
    execute(circ, st, fuse=False)
    out = st.amplitudes()
    st.close()
    return out


@pytest.fixture(autouse=True)
def compiled():
    old = os.environ.get("QSB_FUSED_JIT")
    os.environ["QSB_FUSED_JIT"] = "2"
    yield
    if old is None:
        os.environ.pop("QSB_FUSED_JIT", None)
    else:
        os.environ["QSB_FUSED_JIT"] = old


def test_interleaved_handles():
    n = 20
    circs = [build_qft(n), layered_random_circuit(n, 4, seed=3)]
    a0 = [rand_amps(n, 1), rand_amps(n, 2)]
    refs = [reference(c, a) for c, a in zip(circs, a0)]
    states = []
    for a in a0:
        st = State(n)
        st.set_amplitudes(a)
        states.append(st)
    plans = [fusion.plan(n, lower_ops(c)) for c in circs]
    # pass i of circuit 0, then pass i of circuit 1, ... with no syncs between
    for i in range(max(len(p) for p in plans)):
        for st, p in zip(states, plans):
            if i < len(p):
                fusion.run(st, [p[i]])
    for st, ref in zip(states, refs):
        assert same_values(st.amplitudes(), ref)
        st.close()


def test_recycled_handles():
    n = 19
    circ = build_qft(n)
    a0 = rand_amps(n, 7)
    ref = reference(circ, a0)
    for _ in range(4):  # each handle takes its counter from the cache of the last
        st = State(n)
        st.set_amplitudes(a0)
        execute(circ, st, fuse=True)
        assert same_values(st.amplitudes(), ref)
        st.close()


@pytest.mark.parametrize("q", [13, 14, 19])
def test_unequal_tiles(q):
    """Phases on qubits outside the tile: tiles with the bit set do all the
    work, the others none (tile-index bits 0-1 used to be constant per CTA)."""
    n = 20
    ins = []
    for i in range(40):
        ins.append(Apply(u1(0.05 + 0.01 * i), q))
        ins.append(ControlledApply(u1(0.3 + 0.02 * i), q, 3))
    circ = Circuit(n, tuple(ins))
    a0 = rand_amps(n, q)
    ref = reference(circ, a0)
    st = State(n)
    st.set_amplitudes(a0)
    tile = list(range(12))
    st.apply_fused(tile, fusion.Pass(tile, lower_ops(circ)).op_array())
    assert same_values(st.amplitudes(), ref)
    st.close()
