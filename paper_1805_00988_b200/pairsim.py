"""pairsim-compatible function API backed by the B200 kernels.

Drop-in for the reference's public functions (pkg/src/pairsim/__init__.py:10-88)
so code written against pairsim — including its own tests — can be pointed at
the GPU by swapping the import:

    import paper_1805_00988_b200.pairsim as pairsim

Semantics follow the reference function by function (cited below).  The one
structural difference is where the register lives: ``StateVector.amps`` is a
host mirror of the device buffer.  It is materialised on first access and,
once handed out, kept coherent: it is uploaded before and refreshed after
every device operation, so in-place edits such as ``state.amps[:] = v``
(pkg/tests/test_kernel.py:37) behave exactly as with a numpy-resident
register.  Code that never touches ``.amps`` never pays a host copy.

Both reference precisions live on the device: Precision.SINGLE registers are
complex64, Precision.DOUBLE registers complex128 (gates64.cu), so the
reference's fp64 acceptance criteria (1e-10 vs the dense oracle) apply too.
"""

from __future__ import annotations

import enum
import os

import numpy as np

from . import _native as N
from .circuits import (  # noqa: F401  (re-exported, as pairsim/__init__.py does)
    Apply,
    Circuit,
    ControlledApply,
    ControlledControlledApply,
    SampleMeasure,
    build_bernstein_vazirani,
    build_qft,
    random_circuit,
)
from .errors import (  # noqa: F401
    CapacityError,
    DegenerateStateError,
    DimensionError,
    NotUnitaryError,
    ParseError,
    ValidationError,
)
from .gates import (  # noqa: F401
    FIXED_GATES,
    Gate,
    H,
    S,
    T,
    X,
    Y,
    Z,
    is_unitary,
    make_gate,
    random_unitary_gate,
    std_gate,
    u1,
)
from .qc import format_circuit, parse_circuit  # noqa: F401  (circuits.py:86-168)
from .state import State

MAX_SUPPORTED_QUBITS = 300  # state.py:20


class Precision(enum.Enum):
    """state.py:25-42; SINGLE = complex64, DOUBLE = complex128 in HBM."""

    SINGLE = "single"
    DOUBLE = "double"

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.complex64 if self is Precision.SINGLE else np.complex128)

    @property
    def bits_per_amplitude(self) -> int:
        return 64 if self is Precision.SINGLE else 128

    @property
    def norm_tolerance(self) -> float:
        return 1e-4 if self is Precision.SINGLE else 1e-10


def memory_required(num_qubits: int, precision: Precision = Precision.SINGLE) -> int:
    """Bits for the amplitude array (state.py:71-83)."""
    if num_qubits < 1:
        raise ValueError("num_qubits must be >= 1")
    if num_qubits > MAX_SUPPORTED_QUBITS:
        raise CapacityError(f"{num_qubits} qubits is past the supported limit of {MAX_SUPPORTED_QUBITS}")
    return precision.bits_per_amplitude << num_qubits


def format_bytes(num_bytes: int) -> str:
    """Decimal units, 4 significant digits (state.py:86-97)."""
    if num_bytes < 1000:
        return f"{num_bytes} B"
    value = float(num_bytes)
    unit = "B"
    for unit in ("kB", "MB", "GB", "TB", "PB", "EB"):
        value /= 1000.0
        if value < 1000.0:
            break
    digits = 3 if value < 10 else (2 if value < 100 else 1)
    return f"{f'{value:.{digits}f}'.rstrip('0').rstrip('.')} {unit}"


def default_memory_budget() -> int:
    """0 selects the device default: 75% of free HBM (cf. state.py:114-119)."""
    return 0


def _device() -> int:
    return int(os.environ.get("QSB_DEVICE", "0"))


class _Mirror(np.ndarray):
    """Host copy of a register handed out as `StateVector.amps`.  Every write
    through it — item / slice assignment, in-place operators and ufuncs with
    `out=`, numpy functions with `out=`, ndarray's mutating methods,
    np.copyto / np.put / np.place / np.putmask — marks it dirty (views share
    the flag), so the next device operation uploads it; an untouched mirror
    is not re-uploaded.  (Writes through a plain-ndarray view of it, e.g.
    `amps.view(np.ndarray)`, or through raw pointers are not seen: assign
    `state.amps = array` after such edits.)"""

    _MUTATORS = ("fill", "put", "sort", "partition", "resize", "setfield", "byteswap")

    def __array_finalize__(self, obj):
        self._flag = getattr(obj, "_flag", None)

    def _touch(self):
        if self._flag is not None:
            self._flag[0] = True

    def __setitem__(self, key, value):
        self._touch()
        super().__setitem__(key, value)

    def __array_ufunc__(self, ufunc, method, *inputs, out=None, **kwargs):
        plain = tuple(np.asarray(x) if isinstance(x, _Mirror) else x for x in inputs)
        if out is not None:
            for o in out:
                if isinstance(o, _Mirror):
                    o._touch()
            kwargs["out"] = tuple(np.asarray(o) if isinstance(o, _Mirror) else o for o in out)
        res = getattr(ufunc, method)(*plain, **kwargs)
        if out is not None and len(out) == 1 and isinstance(out[0], _Mirror):
            return out[0]  # in-place operators keep the tracked object
        return res

    def __array_function__(self, func, types, args, kwargs):
        if func in (np.copyto, np.put, np.place, np.putmask, np.fill_diagonal) and args and \
                isinstance(args[0], _Mirror):
            args[0]._touch()
        out = kwargs.get("out")  # np.dot(..., out=amps), np.matmul(..., out=amps), ...
        for o in (out if isinstance(out, tuple) else (out,)):
            if isinstance(o, _Mirror):
                o._touch()
        return super().__array_function__(func, types, args, kwargs)

    def __reduce__(self):  # pickles as a plain array
        return np.asarray(self).__reduce__()


def _mutator(name):
    def method(self, *a, **k):
        if name != "byteswap" or k.get("inplace") or (a and a[0]):
            self._touch()
        return getattr(np.ndarray, name)(self, *a, **k)

    method.__name__ = name
    return method


for _name in _Mirror._MUTATORS:
    setattr(_Mirror, _name, _mutator(_name))


class StateVector:
    """Register handle (state.py:45-68) whose amplitudes live in HBM."""

    def __init__(self, num_qubits: int, amps=None, *, _dev: State | None = None):
        if num_qubits < 1:
            raise ValueError("num_qubits must be >= 1")
        self.num_qubits = int(num_qubits)
        self._mirror: np.ndarray | None = None
        self._dirty = [False]  # the handed-out mirror was written since the last sync
        self._uploads = 0  # host -> device re-uploads of a written mirror (diagnostics)
        if _dev is not None:
            self._dev = _dev
            return
        arr = np.asarray(amps)
        dim = 1 << self.num_qubits
        if arr.shape != (dim,):
            raise ValueError(f"expected {dim} amplitudes, got shape {arr.shape}")
        if arr.dtype not in (np.complex64, np.complex128):
            raise ValueError(f"unsupported amplitude dtype {arr.dtype}")
        self._dev = State(self.num_qubits, _device(), precision=arr.dtype)
        self._dev.set_amplitudes(arr)

    @property
    def dim(self) -> int:
        return 1 << self.num_qubits

    @property
    def precision(self) -> Precision:
        return Precision.DOUBLE if self._dev.is_double else Precision.SINGLE

    @property
    def device_state(self) -> State:
        return self._dev

    @property
    def amps(self) -> np.ndarray:
        if self._mirror is None:
            m = self._dev.amplitudes().view(_Mirror)
            m._flag = self._dirty
            self._dirty[0] = False
            self._mirror = m
        return self._mirror

    @amps.setter
    def amps(self, value) -> None:
        arr = np.asarray(value)
        if arr.shape != (self.dim,) or arr.dtype != self._dev.dtype:
            raise ValueError(f"amps must be a {self._dev.dtype} array of length 2^n")
        if isinstance(value, _Mirror) and value._flag is self._dirty:
            self._mirror = value  # `state.amps op= x` hands the tracked mirror back
        else:
            self._mirror = arr  # a caller's plain array: untracked, so always treated as written
        self._dev.set_amplitudes(arr)
        self._dirty[0] = False

    def _host_written(self) -> bool:
        return not isinstance(self._mirror, _Mirror) or self._dirty[0]

    # device-op bracket: keep a handed-out mirror coherent (upload only what
    # the host wrote; download the result into the same array object)
    def _before(self) -> State:
        if self._mirror is not None and self._host_written():
            self._dev.set_amplitudes(np.asarray(self._mirror))
            self._dirty[0] = False
            self._uploads += 1
        return self._dev

    def _after(self) -> None:
        if self._mirror is not None:
            np.asarray(self._mirror)[:] = self._dev.amplitudes()
            self._dirty[0] = False


def new_state(num_qubits: int, precision: Precision = Precision.SINGLE, memory_budget: int | None = None) -> StateVector:
    """|0...0> on the device; CapacityError before allocation (state.py:122-143)."""
    return _new_state(num_qubits, precision, memory_budget, True)


def _new_state(num_qubits: int, precision: Precision, memory_budget: int | None, init: bool) -> StateVector:
    if num_qubits < 1:
        raise ValueError("num_qubits must be >= 1")
    need = memory_required(num_qubits, precision) // 8
    if memory_budget is not None and need > memory_budget:
        raise CapacityError(
            f"{num_qubits} qubits need {format_bytes(need)} ({need} bytes); "
            f"memory budget is {format_bytes(memory_budget)}")
    dev = State(num_qubits, _device(), memory_budget=memory_budget, precision=precision.value, _init=init)
    return StateVector(num_qubits, _dev=dev)


def norm_squared(state: StateVector) -> float:
    """fp64 sum of |a|^2 (state.py:146-151)."""
    return state._before().norm_squared()


def amplitude_of(state: StateVector, basis_index: int) -> complex:
    """state.py:154-161"""
    if not 0 <= basis_index < state.dim:
        raise IndexError(f"basis index {basis_index} out of range [0, {state.dim})")
    return state._before().amplitude(basis_index)


def nth_cleared(i, target):
    """kernel.py:31-37 (host arithmetic; the device evaluates it in registers)."""
    mask = (1 << target) - 1
    return (i & mask) | ((i & ~mask) << 1)


def apply_gate(state: StateVector, target: int, gate, executor=None) -> StateVector:
    """kernel.py:108-132; `executor` is accepted and ignored (the stream orders sweeps)."""
    n = state.num_qubits
    if not 0 <= target < n:
        raise IndexError(f"target {target} out of range for {n} qubits")
    state._before().apply_gate(gate, target)
    state._after()
    return state


def apply_controlled_gate(state: StateVector, control: int, target: int, gate, executor=None) -> StateVector:
    """kernel.py:135-165 (same validation order)."""
    n = state.num_qubits
    if not 0 <= target < n:
        raise IndexError(f"target {target} out of range for {n} qubits")
    if not 0 <= control < n:
        raise IndexError(f"control {control} out of range for {n} qubits")
    if control == target:
        raise ValueError("control and target must differ")
    state._before().apply_controlled_gate(gate, control, target)
    state._after()
    return state


def apply_controlled_controlled_gate(state: StateVector, control1: int, control2: int, target: int,
                                     gate, executor=None) -> StateVector:
    """QCGPU's doubly-controlled update (no pairsim counterpart)."""
    state._before().apply_controlled_controlled_gate(gate, control1, control2, target)
    state._after()
    return state


class MeasurementHistogram:
    """Counts per basis index for one batch of draws (measure.py:37-65)."""

    def __init__(self, counts: dict[int, int], samples: int):
        self.counts = counts
        self.samples = samples

    def __eq__(self, other):
        return isinstance(other, MeasurementHistogram) and (self.counts, self.samples) == (other.counts, other.samples)

    def __repr__(self):
        return f"MeasurementHistogram(counts={self.counts!r}, samples={self.samples})"

    @classmethod
    def from_outcomes(cls, outcomes: np.ndarray) -> "MeasurementHistogram":
        keys, counts = np.unique(outcomes, return_counts=True)
        # .tolist() gives Python ints in np.unique (sorted) order, 3-4x faster
        # than converting element by element (1e6 distinct outcomes: 240 -> ~70 ms)
        return cls(dict(zip(keys.tolist(), counts.tolist())), int(len(outcomes)))

    def to_csv(self) -> str:
        rows = ["basis_index,count"] + [f"{k},{self.counts[k]}" for k in sorted(self.counts)]
        return "\n".join(rows) + "\n"

    def bar_chart(self, num_qubits: int | None = None, max_width: int = 40) -> str:
        if not self.counts:
            return ""
        peak = max(self.counts.values())
        width = num_qubits if num_qubits is not None else (max(self.counts).bit_length() or 1)
        out = []
        for k in sorted(self.counts):
            c = self.counts[k]
            bar = "#" * max(1, round(max_width * c / peak)) if c else ""
            out.append(f"|{k:0{width}b}>  {c:>8}  {bar}")
        return "\n".join(out)


def probabilities(state: StateVector) -> np.ndarray:
    """fp64 |a|^2, bit-exact (measure.py:29-34)."""
    return state._before().probabilities()


def sample(state: StateVector, n_samples: int, seed: int | None = None) -> MeasurementHistogram:
    """measure.py:76-85; identical histogram for the same seed."""
    if n_samples < 1:
        raise ValueError("n_samples must be >= 1")
    return MeasurementHistogram.from_outcomes(state._before().sample_outcomes(n_samples, seed))


def measure_collapse(state: StateVector, seed: int | None = None) -> tuple[int, StateVector]:
    """measure.py:88-99: one draw, then the register becomes e_outcome exactly."""
    outcome = state._before().measure_collapse(seed)
    state._after()
    return outcome, state


def run_circuit(circuit, precision: Precision = Precision.SINGLE, seed=None, executor=None,
                memory_budget=None, fuse: bool = True):
    """circuits.py:171-192 on the device; returns (StateVector, histogram | None)."""
    from .circuits import execute

    # |0> is written by the circuit's first fused pass (or an explicit reset
    # when it has none): the register is not cleared separately
    state = _new_state(circuit.num_qubits, precision, memory_budget, False)
    outcomes = execute(circuit, state.device_state, seed=seed, fuse=fuse, initial_basis=0)
    hist = MeasurementHistogram.from_outcomes(outcomes) if outcomes is not None else None
    return state, hist
