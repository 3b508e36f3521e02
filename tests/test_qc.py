"""The .qc text format and the command-line front-end.

Parse / format cases are ports of the reference's own tests
(pkg/tests/test_circuits.py:29-113) against paper_1805_00988_b200.qc; the CLI
cases port pkg/tests/test_cli.py:14-80 and run the circuit on the GPU.
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_1805_00988_b200 import cli
from paper_1805_00988_b200.circuits import (
    Apply,
    Circuit,
    ControlledApply,
    ControlledControlledApply,
    SampleMeasure,
    build_qft,
    random_circuit,
)
from paper_1805_00988_b200.errors import ParseError, ValidationError
from paper_1805_00988_b200.gates import H, X, make_gate, u1
from paper_1805_00988_b200.qc import format_circuit, parse_circuit


class TestParse:
    def test_basic_circuit(self):
        c = parse_circuit("qubits 2\nh 0\ncx 0 1")
        assert c.num_qubits == 2
        assert c.instructions == (Apply(H, 0), ControlledApply(X, 0, 1))

    def test_index_out_of_range(self):
        with pytest.raises(ValidationError):
            parse_circuit("qubits 1\nh 5")

    def test_controlled_phase_with_angle(self):
        assert parse_circuit("qubits 2\ncu1 0 1 1.5707963").instructions == (
            ControlledApply(u1(1.5707963), 0, 1),)

    def test_comments_and_blanks_ignored(self):
        text = "# a circuit\nqubits 2\n\nh 0  # superpose\n  \ncx 0 1\n"
        assert parse_circuit(text).instructions == (Apply(H, 0), ControlledApply(X, 0, 1))

    def test_measure_line(self):
        assert parse_circuit("qubits 1\nh 0\nmeasure 500").instructions[-1] == SampleMeasure(500)

    def test_doubly_controlled_extension(self):
        c = parse_circuit("qubits 3\nccx 0 1 2\nccu1 2 0 1 0.5")
        assert c.instructions == (ControlledControlledApply(X, 0, 1, 2),
                                  ControlledControlledApply(u1(0.5), 2, 0, 1))
        assert parse_circuit(format_circuit(c)) == c
        with pytest.raises(ValidationError):
            parse_circuit("qubits 3\nccx 0 0 2")

    @pytest.mark.parametrize("text,line", [
        ("h 0", 1), ("qubits 2\nfoo 0", 2), ("qubits 2\nh zero", 2), ("qubits 2\nu1 0 fast", 2),
        ("qubits 2\nh 0 1", 2), ("qubits 2\nqubits 3", 2), ("qubits 2\nmeasure many", 2),
        ("qubits 3\nccx 0 1", 2),
    ])
    def test_parse_errors_carry_line_numbers(self, text, line):
        with pytest.raises(ParseError) as err:
            parse_circuit(text)
        assert err.value.line_no == line and f"line {line}" in str(err.value)

    @pytest.mark.parametrize("text", ["qubits 2\ncx 1 1", "qubits 2\nmeasure 10\nh 0",
                                      "qubits 2\nmeasure 0", "qubits 0"])
    def test_validation_errors(self, text):
        with pytest.raises(ValidationError):
            parse_circuit(text)

    def test_missing_header_on_empty_text(self):
        with pytest.raises(ParseError):
            parse_circuit("")


class TestFormat:
    def test_single_gate(self):
        assert format_circuit(Circuit(1, (Apply(H, 0),))) == "qubits 1\nh 0"

    def test_qft2_exact_text(self):
        assert format_circuit(build_qft(2)) == "qubits 2\nh 0\ncu1 1 0 1.5707963267948966\nh 1"

    def test_measure_formatted(self):
        assert format_circuit(Circuit(1, (Apply(H, 0), SampleMeasure(100)))).endswith("measure 100")

    def test_custom_gate_not_formattable(self):
        with pytest.raises(ValueError):
            format_circuit(Circuit(1, (Apply(make_gate(np.eye(2)), 0),)))

    def test_round_trip_identity_on_random_circuits(self):
        rng = np.random.default_rng(31)
        for _ in range(100):
            n = int(rng.integers(1, 9))
            c = random_circuit(n, int(rng.integers(1, 25)), rng, custom_fraction=0.0)
            assert parse_circuit(format_circuit(c)) == c


BELL = "qubits 2\nh 0\ncx 0 1\n"


def write(tmp_path, text, name="circuit.qc"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


class TestCliErrors:
    """Paths that fail before any device work (no GPU needed)."""

    def test_bad_gate_name_exits_1_with_line(self, tmp_path, capsys):
        assert cli.main(["run", write(tmp_path, "qubits 1\nfrobnicate 0\n")]) == 1
        cap = capsys.readouterr()
        assert cap.out == "" and "line 2" in cap.err and "kind=ParseError" in cap.err

    def test_missing_file_exits_3(self, capsys):
        assert cli.main(["run", "/nonexistent/x.qc"]) == 3
        assert "kind=FileNotFoundError" in capsys.readouterr().err

    def test_usage_error_exits_1(self, capsys):
        with pytest.raises(SystemExit) as e:
            cli.main(["run"])
        assert e.value.code == 1 and "kind=UsageError" in capsys.readouterr().err


@pytest.mark.gpu
class TestCliOnDevice:
    def test_bell_histogram_hits_only_00_and_11(self, tmp_path, capsys):
        assert cli.main(["run", write(tmp_path, BELL), "--shots", "1000", "--seed", "9"]) == 0
        lines = capsys.readouterr().out.strip().splitlines()
        assert lines[0] == "basis_index,count"
        idx = {int(x.split(",")[0]) for x in lines[1:]}
        assert idx <= {0, 3} and sum(int(x.split(",")[1]) for x in lines[1:]) == 1000

    def test_circuit_measure_line_used_without_shots_flag(self, tmp_path, capsys):
        assert cli.main(["run", write(tmp_path, "qubits 1\nx 0\nmeasure 25\n")]) == 0
        assert "1,25" in capsys.readouterr().out

    def test_chart_flag_prints_bars(self, tmp_path, capsys):
        assert cli.main(["run", write(tmp_path, BELL), "--shots", "200", "--seed", "9", "--chart"]) == 0
        out = capsys.readouterr().out
        assert "|00>" in out and "#" in out

    def test_amplitudes_printed_without_sampling(self, tmp_path, capsys):
        assert cli.main(["run", write(tmp_path, BELL)]) == 0
        out = capsys.readouterr().out
        assert "|00>" in out and "0x0" in out and "p=0.5" in out

    def test_oversized_register_exits_2_with_byte_count(self, tmp_path, capsys):
        assert cli.main(["run", write(tmp_path, "qubits 40\nh 0\n")]) == 2
        err = capsys.readouterr().err
        assert "kind=CapacityError" in err and str((64 << 40) // 8) in err

    def test_determinism_and_fused_equals_unfused(self, tmp_path, capsys):
        text = "qubits 12\n" + "\n".join(f"h {q}" for q in range(12)) + "\ncu1 11 3 0.7\nccx 0 5 9\nmeasure 4000\n"
        path = write(tmp_path, text)
        outs = []
        for flags in (["--seed", "3"], ["--seed", "3"], ["--seed", "3", "--no-fuse"]):
            assert cli.main(["run", path, *flags]) == 0
            outs.append(capsys.readouterr().out)
        assert outs[0] == outs[1] == outs[2]

    def test_state_limit_and_double(self, tmp_path, capsys):
        path = write(tmp_path, "qubits 3\nh 0\nh 1\nh 2\nmeasure 10\n")
        assert cli.main(["state", path, "--limit", "4", "--precision", "double"]) == 0
        out = capsys.readouterr().out.strip().splitlines()
        assert len(out) == 4 and all("0x" in x and "p=0.125000" in x for x in out)

    def test_bv_decodes_hidden_integer(self, capsys):
        assert cli.main(["bv", "14", "101"]) == 0
        out = capsys.readouterr().out
        assert "101: 1000" in out and "decoded: 101" in out
