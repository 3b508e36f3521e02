"""The reference's ``.qc`` circuit text format (pkg/src/pairsim/circuits.py:1-16,
86-168), read into this package's Circuit IR so user circuit files run on the
B200 backend.

    qubits N            header, first non-comment line
    h 0                 gate mnemonic + target            (h x y z s t)
    u1 2 0.785398       parametric gate, trailing angle in radians
    cx 0 1              controlled: control, then target  (ch cx cy cz cs ct cu1)
    ccx 0 1 2           doubly controlled: c1, c2, target (extension: the
                        QCGPU apply_controlled_controlled_gate instructions,
                        which pairsim's format has no spelling for)
    measure 1000        sample count; final instruction only
    # comment           ignored, as are blank lines

Error behaviour follows the reference: ParseError (with the 1-based line
number) for malformed text, ValidationError for well-formed but out-of-
contract circuits (circuits.py:61-80).  ``format_circuit`` emits the
canonical text and ``parse_circuit(format_circuit(c)) == c``.
"""

from __future__ import annotations

from .circuits import Apply, Circuit, ControlledApply, ControlledControlledApply, SampleMeasure
from .errors import ParseError, ValidationError
from .gates import FIXED_GATES, std_gate

_NAMES = set(FIXED_GATES) | {"u1"}


def parse_circuit(text: str) -> Circuit:
    num_qubits = None
    out = []
    for line_no, raw in enumerate(text.splitlines(), start=1):
        line = raw.split("#", 1)[0].strip()
        if not line:
            continue
        word, *args = line.split()
        word = word.lower()
        if num_qubits is None:
            if word != "qubits":
                raise ParseError(line_no, f"expected 'qubits N' header, got {word!r}")
            num_qubits = _one_int(line_no, args, "qubit count")
            if num_qubits < 1:
                raise ValidationError(f"line {line_no}: qubit count must be >= 1")
            continue
        if word == "qubits":
            raise ParseError(line_no, "duplicate 'qubits' header")
        if word == "measure":
            out.append(SampleMeasure(_one_int(line_no, args, "sample count")))
            continue
        out.append(_gate_line(line_no, word, args))
    if num_qubits is None:
        raise ParseError(max(1, text.count("\n") + 1), "missing 'qubits N' header")
    try:
        return Circuit(num_qubits, tuple(out))
    except ValidationError as exc:
        raise ValidationError(f"{exc} (in parsed circuit)") from exc


def _one_int(line_no: int, args, what: str) -> int:
    if len(args) != 1:
        raise ParseError(line_no, f"expected one {what}")
    try:
        return int(args[0])
    except ValueError:
        raise ParseError(line_no, f"{what} must be an integer, got {args[0]!r}") from None


def _gate_line(line_no: int, word: str, args):
    ncontrols = 2 if word.startswith("cc") and word[2:] in _NAMES else (
        1 if word.startswith("c") and word[1:] in _NAMES else 0)
    name = word[ncontrols:]
    if name not in _NAMES:
        raise ParseError(line_no, f"unknown gate {word!r}")
    nq = ncontrols + 1
    want = nq + (1 if name == "u1" else 0)
    if len(args) != want:
        raise ParseError(line_no, f"gate {word!r} expects {want} argument(s)")
    try:
        qubits = [int(a) for a in args[:nq]]
    except ValueError:
        raise ParseError(line_no, f"qubit indices must be integers: {args!r}") from None
    angle = None
    if name == "u1":
        try:
            angle = float(args[-1])
        except ValueError:
            raise ParseError(line_no, f"angle must be a number, got {args[-1]!r}") from None
    gate = std_gate(name, angle)
    if ncontrols == 2:
        return ControlledControlledApply(gate, qubits[0], qubits[1], qubits[2])
    if ncontrols == 1:
        return ControlledApply(gate, qubits[0], qubits[1])
    return Apply(gate, qubits[0])


def format_circuit(circuit: Circuit) -> str:
    """Canonical text for a circuit of library gates (circuits.py:152-168);
    ValueError for gates without a mnemonic."""
    lines = [f"qubits {circuit.num_qubits}"]
    for ins in circuit.instructions:
        if isinstance(ins, SampleMeasure):
            lines.append(f"measure {ins.n_samples}")
            continue
        g = ins.gate
        if g.name not in _NAMES:
            raise ValueError(f"gate {g.name!r} has no text mnemonic")
        angle = f" {g.angle!r}" if g.name == "u1" else ""
        if isinstance(ins, Apply):
            lines.append(f"{g.name} {ins.target}{angle}")
        elif isinstance(ins, ControlledApply):
            lines.append(f"c{g.name} {ins.control} {ins.target}{angle}")
        else:
            lines.append(f"cc{g.name} {ins.control1} {ins.control2} {ins.target}{angle}")
    return "\n".join(lines)
