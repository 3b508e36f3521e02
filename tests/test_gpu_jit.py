"""Run-time compiled fused-pass programs (csrc/jit.cu) against the interpreter
kernel and the oracle.

QSB_FUSED_JIT=2 compiles every pass with NVRTC before launching it, 0 runs the
ahead-of-time interpreter; 1 (the default) queues the compile on a host worker
and interprets the pass until its program is ready.  All must give the same
bits.
"""

from __future__ import annotations

import math
import os
from contextlib import contextmanager

import numpy as np
import pytest

from golden_util import same_values
from oracle import c as oc
from paper_1805_00988_b200 import (
    State,
    build_hadamard_layer,
    build_qft,
    execute,
    layered_random_circuit,
    random_circuit,
    random_unitary_gate,
    u1,
)
from paper_1805_00988_b200.circuits import Apply, Circuit, ControlledApply, ControlledControlledApply
from paper_1805_00988_b200.gates import FIXED_GATES

pytestmark = pytest.mark.gpu


@contextmanager
def jit(mode):
    old = os.environ.get("QSB_FUSED_JIT")
    os.environ["QSB_FUSED_JIT"] = str(mode)
    try:
        yield
    finally:
        if old is None:
            os.environ.pop("QSB_FUSED_JIT", None)
        else:
            os.environ["QSB_FUSED_JIT"] = old


def rand_amps(n, rng):
    v = rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)
    return (v / np.linalg.norm(v)).astype(np.complex64)


def run(circ, a0, mode, K=None, rb="4"):
    old = os.environ.get("QSB_FUSED_RB")
    os.environ["QSB_FUSED_RB"] = rb
    try:
        with jit(mode):
            st = State(circ.num_qubits)
            st.set_amplitudes(a0)
            execute(circ, st, fuse=True, tile_qubits=K)
            return st.amplitudes()
    finally:
        if old is None:
            os.environ.pop("QSB_FUSED_RB", None)
        else:
            os.environ["QSB_FUSED_RB"] = old


def mixed(n, count, rng):
    lib = list(FIXED_GATES.values())
    ins = []
    for _ in range(count):
        t = int(rng.integers(n))
        r = rng.random()
        g = (random_unitary_gate(rng) if r < 0.3 else u1(float(rng.uniform(0, 2 * math.pi))) if r < 0.5
             else lib[int(rng.integers(len(lib)))])
        others = [q for q in range(n) if q != t]
        k = rng.random()
        if k < 0.5:
            ins.append(Apply(g, t))
        elif k < 0.85:
            ins.append(ControlledApply(g, int(rng.choice(others)), t))
        else:
            c1, c2 = (int(x) for x in rng.choice(others, 2, replace=False))
            ins.append(ControlledControlledApply(g, c1, c2, t))
    return Circuit(n, tuple(ins))


@pytest.mark.parametrize("name,n", [("hlayer", 20), ("qft", 18), ("qft", 24), ("layered", 22), ("mixed", 16)])
def test_compiled_equals_interpreted(name, n):
    rng = np.random.default_rng(1000 + n)
    a0 = rand_amps(n, rng)
    circ = {"hlayer": lambda: build_hadamard_layer(n), "qft": lambda: build_qft(n),
            "layered": lambda: layered_random_circuit(n, 4, seed=n),
            "mixed": lambda: mixed(n, 150, rng)}[name]()
    interp = run(circ, a0, 0)
    compiled = run(circ, a0, 2)
    assert same_values(interp, compiled)


@pytest.mark.parametrize("rb", ["3", "4"])
@pytest.mark.parametrize("K", [10, 12, 13])
def test_compiled_vs_oracle_all_tile_shapes(K, rb):
    n = 15
    rng = np.random.default_rng(77 + K)
    a0 = rand_amps(n, rng)
    circ = mixed(n, 90, rng)
    ref = a0.copy()
    for i in circ.instructions:
        if isinstance(i, Apply):
            oc.apply_gate(ref, i.target, i.gate)
        elif isinstance(i, ControlledApply):
            oc.apply_controlled_gate(ref, i.control, i.target, i.gate)
        else:
            oc.apply_cc_gate(ref, i.control1, i.control2, i.target, i.gate)
    assert same_values(run(circ, a0, 2, K=K, rb=rb), ref)


def test_background_compile_policy():
    """Mode 1 (default): a pass's first launches are interpreted while its
    program compiles on a host worker; after qs_jit_sync the compiled program
    runs.  The register evolves identically either way."""
    from paper_1805_00988_b200 import fusion

    n = 19
    rng = np.random.default_rng(5)
    a0 = rand_amps(n, rng)
    circ = build_qft(n)
    with jit(1):
        st = State(n)
        st.set_amplitudes(a0)
        execute(circ, st, fuse=True)
        fusion.jit_sync()
        for _ in range(2):
            execute(circ, st, fuse=True)
        got = st.amplitudes()
    with jit(0):
        ref = State(n)
        ref.set_amplitudes(a0)
        for _ in range(3):
            execute(circ, ref, fuse=True)
        assert same_values(got, ref.amplitudes())


def test_program_disk_cache_across_processes(tmp_path):
    """A second process running the same fused circuit loads the compiled
    pass programs from the on-disk cache (no NVRTC), with the same bits."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    child = (
        "import sys, json, numpy as np\n"
        f"sys.path.insert(0, {str(root)!r})\n"
        "from paper_1805_00988_b200 import State, build_qft, fusion\n"
        "from paper_1805_00988_b200.circuits import lower_ops\n"
        "st = State(16)\n"
        "for q in range(16): st.h(q)\n"
        "fusion.run(st, fusion.plan(16, lower_ops(build_qft(16)), 11))\n"
        "a = st.amplitudes()\n"
        "print(json.dumps({**fusion.jit_stats(), 'digest': a.tobytes().hex()[:64] + str(float(np.abs(a).sum()))}))\n")
    env = dict(__import__("os").environ, QSB_JIT_CACHE_DIR=str(tmp_path), QSB_FUSED_JIT="2")
    outs = []
    for _ in range(2):
        r = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0]["compiled"] >= 1 and outs[0]["cache_hits"] == 0
    assert outs[1]["compiled"] == 0 and outs[1]["cache_hits"] == outs[0]["compiled"]
    assert outs[0]["digest"] == outs[1]["digest"]
    assert any(p.suffix == ".bin" for p in tmp_path.iterdir())


def test_parametric_programs_reuse_structure(tmp_path):
    """Circuits with the same structure and other angles (a variational loop):
    the second distinct literal program of a structure switches it to its
    parametric program (entries read from the op table), and every later
    circuit of that structure compiles nothing.  Bits equal the sweeps."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    child = (
        "import sys, json, math, numpy as np\n"
        f"sys.path.insert(0, {str(root)!r})\n"
        "from paper_1805_00988_b200 import State, fusion, u1, execute\n"
        "from paper_1805_00988_b200.circuits import Apply, ControlledApply, Circuit, lower_ops\n"
        "from paper_1805_00988_b200.gates import H\n"
        "n = 16\n"
        "def circ(th):\n"
        "    ins = [Apply(H, q) for q in range(n)]\n"
        "    ins += [ControlledApply(u1(th * (j + 1) / (k + 2)), j, k) for j in range(n) for k in range(j)]\n"
        "    ins += [Apply(H, q) for q in range(n)]\n"
        "    return Circuit(n, tuple(ins))\n"
        "out = []\n"
        "for th in (0.3, 0.7, 1.1, 1.9):\n"
        "    before = fusion.jit_stats()['compiled']\n"
        "    a, b = State(n), State(n)\n"
        "    c = circ(th)\n"
        "    fusion.run(a, fusion.plan(n, lower_ops(c), 11))\n"
        "    execute(c, b, fuse=False)\n"
        "    out.append({'new': fusion.jit_stats()['compiled'] - before,\n"
        "                'same': bool(np.all(a.amplitudes() == b.amplitudes()))})\n"
        "print(json.dumps(out))\n")
    env = dict(__import__("os").environ, QSB_JIT_CACHE="0", QSB_FUSED_JIT="2")
    r = subprocess.run([sys.executable, "-c", child], env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert all(o["same"] for o in out)
    assert out[0]["new"] >= 1 and out[1]["new"] >= 1  # literal, then the parametric programs
    assert out[2]["new"] == 0 and out[3]["new"] == 0


@pytest.mark.parametrize("env", [{"QSB_JIT_STATIC_STAGES": "0"}, {"QSB_JIT_PHASE": "1", "QSB_JIT_LOOP_FORM": "cs"},
                                 {"QSB_FUSED_RUN_BOXES": "0"}])
def test_program_variants_same_bits(tmp_path, env):
    """Code-generation variants kept as switches (the generic stage loop
    instead of the literal-layout one, the scalar phase forms, one-bit TMA box
    dims) give the default programs' bits: each runs a QFT and a layered
    circuit in a fresh process (the switches are read once per process)."""
    import json
    import subprocess
    import sys
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    child = (
        "import sys, json, hashlib\n"
        f"sys.path.insert(0, {str(root)!r})\n"
        "from paper_1805_00988_b200 import State, build_qft, layered_random_circuit, fusion\n"
        "from paper_1805_00988_b200.circuits import lower_ops\n"
        "st = State(18)\n"
        "for q in range(18): st.h(q)\n"
        "fusion.run(st, fusion.plan(18, lower_ops(build_qft(18)), 12))\n"
        "fusion.run(st, fusion.plan(18, lower_ops(layered_random_circuit(18, 4, seed=5)), 12))\n"
        "print(json.dumps({'d': hashlib.sha256(st.amplitudes().tobytes()).hexdigest(), **fusion.jit_stats()}))\n")
    outs = []
    for e in ({}, env):
        full = dict(__import__("os").environ, QSB_JIT_CACHE_DIR=str(tmp_path / str(len(outs))), QSB_FUSED_JIT="2",
                    **e)
        r = subprocess.run([sys.executable, "-c", child], env=full, capture_output=True, text=True, timeout=900)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(json.loads(r.stdout.strip().splitlines()[-1]))
    assert outs[0]["failed"] == 0 and outs[1]["failed"] == 0 and outs[1]["compiled"] >= 1
    assert outs[0]["d"] == outs[1]["d"]


class TestFromBasis:
    """qs_apply_fused_from_basis / execute(..., initial_basis=b): the reset is
    folded into the first fused pass (tiles written as |b>, not loaded).  The
    register must equal reset(b) + the same passes bit for bit, whatever it
    held before (filled with noise here), for bases inside every kind of tile
    position, on the compiled programs and the interpreter, and through the
    fallbacks (small registers, complex128)."""

    @pytest.mark.parametrize("n,circ_name", [(12, "qft"), (16, "layered"), (20, "hlayer"), (20, "qft"),
                                             (21, "random")])
    @pytest.mark.parametrize("jit", ["2", "0"])
    def test_equals_reset_then_passes(self, n, circ_name, jit, monkeypatch):
        from paper_1805_00988_b200 import build_hadamard_layer, layered_random_circuit, random_circuit

        monkeypatch.setenv("QSB_FUSED_JIT", jit)
        rng = np.random.default_rng(n)
        circ = {"qft": lambda: build_qft(n), "layered": lambda: layered_random_circuit(n, 4, seed=3),
                "hlayer": lambda: build_hadamard_layer(n),
                "random": lambda: random_circuit(n, 12, np.random.default_rng(5))}[circ_name]()
        noise = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)).astype(np.complex64)
        for b in (0, (1 << n) - 1, int(rng.integers(0, 1 << n)), 1 << (n - 1), 37):
            ref = State(n)
            ref.set_amplitudes(noise)
            ref.reset(b)
            execute(circ, ref, fuse=True)
            got = State(n)
            got.set_amplitudes(noise)
            execute(circ, got, fuse=True, initial_basis=b)
            assert got.amplitudes().tobytes() == ref.amplitudes().tobytes(), (n, circ_name, b)
            ref.close()
            got.close()

    def test_small_double_and_errors(self):
        for n, prec in ((8, "single"), (14, "double")):
            circ = build_qft(n)
            ref = State(n, precision=prec)
            ref.reset(5)
            execute(circ, ref, fuse=True)
            got = State(n, precision=prec)
            got.set_amplitudes(np.ones(1 << n))
            execute(circ, got, fuse=True, initial_basis=5)
            assert got.amplitudes().tobytes() == ref.amplitudes().tobytes()
        st = State(12)
        with pytest.raises(IndexError):
            execute(build_qft(12), st, initial_basis=1 << 12)
        st.close()


def test_from_basis_inexact_mode():
    """initial_basis with exact=False (reordered passes, combined diagonal
    runs): equal to reset + the same inexact run bit for bit (same programs),
    and to the exact result within the north_star tolerance."""
    n = 20
    circ = Circuit(n, build_hadamard_layer(n).instructions + build_qft(n).instructions)
    ref = State(n)
    ref.reset(3)
    execute(circ, ref, exact=False)
    got = State(n)
    got.set_amplitudes(np.ones(1 << n, np.complex64))
    execute(circ, got, exact=False, initial_basis=3)
    assert got.amplitudes().tobytes() == ref.amplitudes().tobytes()
    ex = State(n)
    ex.reset(3)
    execute(circ, ex)
    want = ex.amplitudes()
    # this state concentrates its weight (|a| up to 0.64) and cancels to ~0
    # elsewhere: the absolute floor scales with the largest amplitude
    np.testing.assert_allclose(got.amplitudes(), want, rtol=1e-5, atol=1e-5 * float(np.abs(want).max()))
    for s in (ref, got, ex):
        s.close()


class TestChunkSumEpilogue:
    """A measured circuit's last fused pass leaves the sampler's chunk sums
    (qs_sample_prepare + QS_FUSED_CHUNK_SUMS) and the sample skips M1.  The
    sums only seed guesses, so draws must equal the plain path's bit for bit
    — also when the sums are stale (the register changed after the pass)."""

    @pytest.mark.parametrize("n,circ_name", [(12, "qft"), (17, "hlayer"), (20, "random"), (22, "layered")])
    @pytest.mark.parametrize("jit", ["2", "0"])
    def test_draws_equal_plain_path(self, n, circ_name, jit, monkeypatch):
        from paper_1805_00988_b200.circuits import SampleMeasure

        monkeypatch.setenv("QSB_FUSED_JIT", jit)
        base = {"qft": lambda: build_qft(n), "hlayer": lambda: build_hadamard_layer(n),
                "random": lambda: random_circuit(n, 10, np.random.default_rng(n)),
                "layered": lambda: layered_random_circuit(n, 5, seed=n)}[circ_name]()
        measured = Circuit(n, base.instructions + (SampleMeasure(4000),))
        got = State(n)
        got_out = execute(measured, got, seed=11, initial_basis=0)
        ref = State(n)
        execute(base, ref)
        want_out = ref.sample_outcomes(4000, 11)
        assert np.array_equal(got_out, want_out)
        assert got.amplitudes().tobytes() == ref.amplitudes().tobytes()
        got.close()
        ref.close()

    def test_stale_sums_still_exact(self):
        from paper_1805_00988_b200 import fusion
        from paper_1805_00988_b200.circuits import lower_ops

        n = 18
        st = State(n)
        st.sample_prepare(3000)
        fusion.run(st, fusion.plan(n, lower_ops(build_qft(n))), chunk_sums=True)
        st.h(3)  # the register changes after the sums were left
        st.t(17)
        got = st.sample_outcomes(3000, 5, sums_ready=True)
        ref = State(n)
        execute(build_qft(n), ref)
        ref.h(3)
        ref.t(17)
        assert np.array_equal(got, ref.sample_outcomes(3000, 5))
        st.close()
        ref.close()


@pytest.mark.parametrize("n", [8, 14, 20])
def test_run_circuit_on_an_uncleared_register(n):
    """pairsim.run_circuit creates its register without the clear
    (qs_create_uninit) and lets the first fused pass write |0> (or resets when
    the circuit has no fused pass): results equal new_state + the sweeps, for
    circuits with and without fused passes and for complex128."""
    from paper_1805_00988_b200 import pairsim as ps
    from paper_1805_00988_b200.circuits import SampleMeasure

    # dirty the pool's cached buffers first, so an uncleared register would show
    for _ in range(2):
        junk = State(n)
        junk.set_amplitudes(np.full(1 << n, 0.5 + 0.25j, np.complex64))
        junk.close()
    cases = [build_qft(n), Circuit(n, (Apply(FIXED_GATES["h"], 1),)), Circuit(n, ()),
             Circuit(n, build_hadamard_layer(n).instructions + (SampleMeasure(500),))]
    for circ in cases:
        for prec in (ps.Precision.SINGLE, ps.Precision.DOUBLE):
            got, hist = ps.run_circuit(circ, prec, seed=3)
            ref = ps.new_state(n, prec)
            execute(Circuit(n, tuple(i for i in circ.instructions if not isinstance(i, SampleMeasure))),
                    ref.device_state, fuse=False)
            assert np.array_equal(ps.probabilities(got), ps.probabilities(ref)), (circ.gate_count(), prec)
            if hist is not None:
                assert hist == ps.sample(ref, 500, 3)
