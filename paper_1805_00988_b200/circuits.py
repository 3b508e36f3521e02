"""Circuit IR, workload builders and device execution.

IR and builders mirror pkg/src/pairsim/circuits.py:33-255 (same instruction
types, same validation, same gate order for build_qft / build_bernstein_vazirani,
same RNG consumption in random_circuit so a seed yields the same circuit), plus
ControlledControlledApply for QCGPU's doubly-controlled gates.

:func:`execute` runs a circuit on a device State: the gate sequence is lowered
to C-ABI ops and grouped into fused passes (fusion.py) — or, with
``fuse=False``, one sweep per gate exactly like run_circuit (circuits.py:171-192).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from typing import Union

import numpy as np

from . import fusion
from .errors import ValidationError
from .gates import FIXED_GATES, H, X, Z, Gate, random_unitary_gate, u1


@dataclass(frozen=True)
class Apply:
    gate: Gate
    target: int


@dataclass(frozen=True)
class ControlledApply:
    gate: Gate
    control: int
    target: int


@dataclass(frozen=True)
class ControlledControlledApply:
    gate: Gate
    control1: int
    control2: int
    target: int


@dataclass(frozen=True)
class SampleMeasure:
    n_samples: int


Instruction = Union[Apply, ControlledApply, ControlledControlledApply, SampleMeasure]


def _qubits(ins) -> tuple[int, ...]:
    if isinstance(ins, Apply):
        return (ins.target,)
    if isinstance(ins, ControlledApply):
        return (ins.control, ins.target)
    return (ins.control1, ins.control2, ins.target)


@dataclass(frozen=True)
class Circuit:
    """Ordered instructions over a fixed register width (circuits.py:54-83)."""

    num_qubits: int
    instructions: tuple

    def __post_init__(self):
        object.__setattr__(self, "instructions", tuple(self.instructions))
        if self.num_qubits < 1:
            raise ValidationError("num_qubits must be >= 1")
        last = len(self.instructions) - 1
        for pos, ins in enumerate(self.instructions):
            if isinstance(ins, SampleMeasure):
                if pos != last:
                    raise ValidationError("measure is only allowed as the final instruction")
                if ins.n_samples < 1:
                    raise ValidationError("measure needs a positive sample count")
                continue
            qs = _qubits(ins)
            for q in qs:
                if not 0 <= q < self.num_qubits:
                    raise ValidationError(f"qubit index {q} out of range for {self.num_qubits} qubits")
            if len(set(qs)) != len(qs):
                raise ValidationError("control and target must differ")

    def gate_count(self) -> int:
        return sum(1 for i in self.instructions if not isinstance(i, SampleMeasure))


def build_qft(num_qubits: int) -> Circuit:
    """For each j: cu1(pi/2^(j-k)) with control j, target k < j, then H(j);
    no trailing swaps (circuits.py:195-210)."""
    if num_qubits < 1:
        raise ValueError("num_qubits must be >= 1")
    ins = []
    for j in range(num_qubits):
        ins.extend(ControlledApply(u1(math.pi / 2 ** (j - k)), j, k) for k in range(j))
        ins.append(Apply(H, j))
    return Circuit(num_qubits, tuple(ins))


def build_hadamard_layer(num_qubits: int) -> Circuit:
    return Circuit(num_qubits, tuple(Apply(H, q) for q in range(num_qubits)))


def build_bernstein_vazirani(num_qubits: int, hidden: int, shots: int = 1000) -> Circuit:
    """H layer, Z on the hidden bits, H layer, measure (circuits.py:213-226)."""
    if not 0 <= hidden < (1 << num_qubits):
        raise ValueError(f"hidden integer {hidden} does not fit in {num_qubits} qubits")
    ins = [Apply(H, q) for q in range(num_qubits)]
    ins += [Apply(Z, q) for q in range(num_qubits) if (hidden >> q) & 1]
    ins += [Apply(H, q) for q in range(num_qubits)]
    ins.append(SampleMeasure(shots))
    return Circuit(num_qubits, tuple(ins))


def random_circuit(num_qubits: int, depth: int, rng: np.random.Generator,
                   controlled_fraction: float = 0.4, custom_fraction: float = 0.25) -> Circuit:
    """Random library / Haar / u1 gate mix; consumes `rng` exactly as
    circuits.py:229-255 does, so equal seeds give equal circuits."""
    library = list(FIXED_GATES.values())
    ins = []
    for _ in range(depth):
        r = rng.random()
        if r < custom_fraction:
            gate = random_unitary_gate(rng)
        elif r < custom_fraction + 0.15:
            gate = u1(float(rng.uniform(0, 2 * math.pi)))
        else:
            gate = library[int(rng.integers(len(library)))]
        target = int(rng.integers(num_qubits))
        if num_qubits > 1 and rng.random() < controlled_fraction:
            control = int(rng.integers(num_qubits - 1))
            control += control >= target
            ins.append(ControlledApply(gate, control, target))
        else:
            ins.append(Apply(gate, target))
    return Circuit(num_qubits, tuple(ins))


def layered_random_circuit(num_qubits: int, depth: int, seed: int) -> Circuit:
    """BASELINE config 4 workload: per layer, H or T on every
    qubit (p = 1/2 each, seeded), then CX on floor(n/2) random disjoint pairs."""
    rng = np.random.default_rng(seed)
    T = FIXED_GATES["t"]
    ins = []
    for _ in range(depth):
        for q in range(num_qubits):
            ins.append(Apply(H if rng.random() < 0.5 else T, q))
        perm = rng.permutation(num_qubits)
        for k in range(num_qubits // 2):
            ins.append(ControlledApply(X, int(perm[2 * k]), int(perm[2 * k + 1])))
    return Circuit(num_qubits, tuple(ins))


def lower_ops(circuit: Circuit, double: bool = False) -> list:
    """(kind, target, ctrl_mask, m) per gate instruction; m holds the entries
    rounded to the register precision (float32, or float64 when `double`)."""
    ops = []
    for ins in circuit.instructions:
        if isinstance(ins, Apply):
            ops.append(fusion.lower(ins.gate, ins.target, (), double))
        elif isinstance(ins, ControlledApply):
            ops.append(fusion.lower(ins.gate, ins.target, (ins.control,), double))
        elif isinstance(ins, ControlledControlledApply):
            ops.append(fusion.lower(ins.gate, ins.target, (ins.control1, ins.control2), double))
    return ops


def execute(circuit: Circuit, state, seed=None, fuse: bool = True, tile_qubits: int | None = None,
            reorder: bool | None = None, exact: bool = True, initial_basis: int | None = None):
    """Apply `circuit` to a device State in place; returns the per-draw outcomes
    of a trailing SampleMeasure (or None).

    exact=True (default): the reference's arithmetic bit for bit.
    exact=False: results equal the reference to rounding (tested at the
    north_star rtol 1e-5), faster: the fused planner may exchange gates on
    disjoint qubits (reorder) and compiled passes combine runs of diagonal
    gates into one product per amplitude (QS_FUSED_COMBINE_PHASES).
    reorder alone (default: QSB_FUSE_REORDER == "1") enables only the first.
    initial_basis=b: start from |b> (pairsim's new_state + run_circuit); with
    fuse=True the reset is folded into the first fused pass (its tiles are
    written as |b> instead of loaded), same bits as state.reset(b) first."""
    if circuit.num_qubits != state.num_qubits:
        raise ValueError("circuit and state widths differ")
    double = getattr(state, "is_double", False)
    ops = lower_ops(circuit, double=double)
    last = circuit.instructions[-1] if circuit.instructions else None
    measured = isinstance(last, SampleMeasure)
    sums = False
    if fuse:
        if double and tile_qubits is None:
            tile_qubits = 12  # complex128 tiles: 2^12 amplitudes = 64 KiB
        if reorder is None:
            import os

            reorder = os.environ.get("QSB_FUSE_REORDER") == "1" or not exact
        passes = fusion.plan(state.num_qubits, ops, tile_qubits, reorder=reorder)
        # a trailing measurement: the last fused pass leaves the sampler's
        # chunk sums as it writes the register back (one read less)
        want_sums = measured and not double and hasattr(state, "sample_prepare")
        if want_sums:
            state.sample_prepare(last.n_samples)
        sums = fusion.run(state, passes, combine=not exact and not double, from_basis=initial_basis,
                          chunk_sums=want_sums)
    else:
        if initial_basis is not None:
            state.reset(int(initial_basis))
        for kind, t, cm, m in ops:
            fusion._single(state, kind, t, cm, m)
    if measured:
        if sums:
            return state.sample_outcomes(last.n_samples, seed, sums_ready=True)
        return state.sample_outcomes(last.n_samples, seed)
    return None
