"""B200-native state-vector backend for the QCGPU / pairsim hot path.

Public surface:
  * :class:`State` — QCGPU-style register in HBM
  * :mod:`paper_1805_00988_b200.pairsim` — pairsim-compatible function API
  * circuits / fusion — IR, builders and the fused-pass planner
  * sharded — registers sharded over P GPUs on their top log2(P) qubits
  * qc / cli — the reference's .qc text format and run/state/bv front-end

All compute runs in libqsb200.so (hand-written sm_100a CUDA behind the C ABI
in include/qsb200.h); there is no CPU fallback.
"""

from .errors import CapacityError, DegenerateStateError, DeviceError, NotUnitaryError  # noqa: F401
from .gates import FIXED_GATES, Gate, H, S, T, X, Y, Z, make_gate, random_unitary_gate, u1  # noqa: F401
from .state import State  # noqa: F401
from .circuits import (  # noqa: F401
    Apply,
    Circuit,
    ControlledApply,
    ControlledControlledApply,
    SampleMeasure,
    build_bernstein_vazirani,
    build_hadamard_layer,
    build_qft,
    execute,
    layered_random_circuit,
    random_circuit,
)

from .qc import format_circuit, parse_circuit  # noqa: F401

__version__ = "0.1.0"
