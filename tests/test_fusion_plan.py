"""Pass planner invariants (CPU): every op lands in exactly one pass, every
pair target is a tile qubit of its pass, ops sharing a qubit keep their
circuit order (the only reordering is of permutation ops past disjoint-qubit
ops, which commutes bit for bit), and tiles hold qubits 0..5 plus K-6 more."""

from __future__ import annotations

import numpy as np
import pytest

from paper_1805_00988_b200 import _native as N
from paper_1805_00988_b200 import build_hadamard_layer, build_qft, fusion, layered_random_circuit, random_circuit
from paper_1805_00988_b200.circuits import lower_ops


def check(n, ops, passes, K):
    flat = [o for p in passes for o in p.ops]
    assert sorted(map(id, flat)) == sorted(map(id, ops))
    pos = {id(o): i for i, o in enumerate(flat)}
    for p in passes:
        assert len(p.tile) == K and set(range(6)) <= set(p.tile)
        for kind, t, _, _ in p.ops:
            if kind == N.QS_OP_PAIR:
                assert t in p.tile
    masks = [(o[2] | (1 << o[1]), pos[id(o)]) for o in ops]
    perm = [o[0] == N.QS_OP_PAIR and fusion.is_permutation(o[3]) for o in ops]
    for i in range(len(ops)):
        for j in range(i + 1, len(ops)):
            if masks[i][1] > masks[j][1]:  # swapped: disjoint, and one of them a permutation
                assert not (masks[i][0] & masks[j][0]), (i, j)
                assert perm[i] or perm[j], (i, j)


@pytest.mark.parametrize("K", [12, 13])
@pytest.mark.parametrize("name", ["layered", "random", "qft", "hlayer"])
def test_plan_invariants(name, K):
    n = 22
    circ = {"layered": lambda: layered_random_circuit(n, 6, seed=3),
            "random": lambda: random_circuit(n, 400, np.random.default_rng(9)),
            "qft": lambda: build_qft(n), "hlayer": lambda: build_hadamard_layer(n)}[name]()
    ops = lower_ops(circ)
    check(n, ops, fusion._plan(n, ops, K), K)


def test_deferral_reduces_passes_on_layered_circuits():
    ops = lower_ops(layered_random_circuit(32, 20, seed=32))
    assert len(fusion._plan(32, ops, 12)) < len(fusion._plan(32, ops, 12, defer=False))


def check_reorder(n, ops, passes, K):
    """The commutation-aware plan: every op once, pair targets in the tile,
    and each qubit's op sequence unchanged (only disjoint ops swap)."""
    flat = [o for p in passes for o in p.ops]
    assert sorted(map(id, flat)) == sorted(map(id, ops))
    for p in passes:
        assert len(p.tile) == K and set(range(6)) <= set(p.tile)
        for kind, t, _, _ in p.ops:
            if kind == N.QS_OP_PAIR:
                assert t in p.tile
    for q in range(n):
        seq_c = [id(o) for o in ops if (o[2] | (1 << o[1])) >> q & 1]
        seq_p = [id(o) for o in flat if (o[2] | (1 << o[1])) >> q & 1]
        assert seq_c == seq_p, q


@pytest.mark.parametrize("K", [12, 13])
@pytest.mark.parametrize("name", ["layered", "random", "qft"])
def test_reorder_plan_invariants(name, K):
    n = 22
    circ = {"layered": lambda: layered_random_circuit(n, 8, seed=4),
            "random": lambda: random_circuit(n, 400, np.random.default_rng(19)),
            "qft": lambda: build_qft(n)}[name]()
    ops = lower_ops(circ)
    check_reorder(n, ops, fusion._plan_reorder(n, ops, K), K)


def test_reorder_cuts_config4_passes():
    """BASELINE config 4 (32 qubits, 960 gates): the in-order planner needs 80
    passes; the commutation-aware one at most 40."""
    ops = lower_ops(layered_random_circuit(32, 20, seed=32))
    assert len(fusion._plan(32, ops, 12)) == 80
    assert len(fusion.plan(32, ops, reorder=True)) <= 40


def test_reordered_sequence_matches_oracle_to_tolerance():
    """Reordering changes rounding only: the reordered op sequence applied by
    the oracle agrees with the circuit order to the north_star rtol 1e-5."""
    from golden_util import M8Gate
    from oracle import c as oc

    n = 14
    circ = layered_random_circuit(n, 10, seed=8)
    ops = lower_ops(circ)
    passes = fusion._plan_reorder(n, ops, 10)

    def run(seq):
        a = np.zeros(1 << n, np.complex64)
        a[0] = 1
        for kind, t, cm, m in seq:
            ctrls = [q for q in range(n) if (cm >> q) & 1]
            g = M8Gate(m)
            if not ctrls:
                oc.apply_gate(a, t, g)
            else:
                oc.apply_controlled_gate(a, ctrls[0], t, g)
        return a

    ref, got = run(ops), run([o for p in passes for o in p.ops])
    np.testing.assert_allclose(got, ref, rtol=1e-5, atol=1e-5 * 2.0 ** (-n / 2))
