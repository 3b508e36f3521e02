"""Generate tests/golden/pairsim_golden.npz from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

Every array below is produced by importing pairsim from
/root/reference/pkg/src and calling its public API; the GPU box has no
/root/reference, so the parity tests there read only the committed .npz.
Large outputs are stored as SHA-256 digests of canonicalised bytes
(amplitudes + 0.0f folds -0 into +0; every other value is unchanged).
"""

from __future__ import annotations

import hashlib
import math
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "pairsim_golden.npz"

sys.path.insert(0, str(REF_SRC))
import pairsim  # noqa: E402
from pairsim import (  # noqa: E402
    H,
    S,
    T,
    X,
    Y,
    Z,
    Apply,
    ControlledApply,
    Precision,
    SerialExecutor,
    apply_controlled_gate,
    apply_gate,
    build_bernstein_vazirani,
    build_qft,
    measure_collapse,
    new_state,
    probabilities,
    random_circuit,
    random_unitary_gate,
    run_circuit,
    sample,
    u1,
)

SER = SerialExecutor()


def m8(gate) -> np.ndarray:
    vals = [np.complex64(complex(x)) for x in (gate.a, gate.b, gate.c, gate.d)]
    return np.array([v for c in vals for v in (c.real, c.imag)], dtype=np.float32)


def digest(arr: np.ndarray) -> str:
    if arr.dtype in (np.complex64, np.float32, np.complex128, np.float64):
        arr = arr + arr.dtype.type(0)  # canonical zero sign
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def random_state(n, rng):
    st = new_state(n, Precision.SINGLE)
    v = rng.normal(size=st.dim) + 1j * rng.normal(size=st.dim)
    st.amps[:] = (v / np.linalg.norm(v)).astype(np.complex64)
    return st


def library_gate(rng):
    lib = [H, X, Y, Z, S, T]
    r = rng.random()
    if r < 0.35:
        return random_unitary_gate(rng)
    if r < 0.5:
        return u1(float(rng.uniform(0, 2 * math.pi)))
    return lib[int(rng.integers(len(lib)))]


def trace(n, n_ops, rng, controlled_fraction=0.4):
    """Random op trace with a snapshot after every op (kind 0 apply, 1 controlled)."""
    st = random_state(n, rng)
    states = [st.amps.copy()]
    ops, mats = [], []
    for k in range(n_ops):
        gate = library_gate(rng)
        t = k % n if k < n else int(rng.integers(n))  # every target at least once
        if n > 1 and rng.random() < controlled_fraction:
            c = int(rng.integers(n - 1))
            c += c >= t
            apply_controlled_gate(st, c, t, gate, SER)
            ops.append((1, c, -1, t))
        else:
            apply_gate(st, t, gate, SER)
            ops.append((0, -1, -1, t))
        mats.append(m8(gate))
        states.append(st.amps.copy())
    return np.array(ops, np.int32), np.array(mats, np.float32), np.array(states)


def circuit_arrays(circuit):
    ops, mats = [], []
    for ins in circuit.instructions:
        if isinstance(ins, Apply):
            ops.append((0, -1, -1, ins.target))
        elif isinstance(ins, ControlledApply):
            ops.append((1, ins.control, -1, ins.target))
        else:
            continue
        mats.append(m8(ins.gate))
    return np.array(ops, np.int32).reshape(-1, 4), np.array(mats, np.float32).reshape(-1, 8)


def prep_basis(n, x):
    st = new_state(n, Precision.SINGLE)
    for q in range(n):
        if (x >> q) & 1:
            apply_gate(st, q, X)
    return st


def prep_entangled(n):
    """H+T layer then a CX chain: an input on which QFT phases are non-trivial."""
    st = new_state(n, Precision.SINGLE)
    for q in range(n):
        apply_gate(st, q, H)
        apply_gate(st, q, T)
    for q in range(n - 1):
        apply_controlled_gate(st, q, q + 1, X)
    return st


def run_qft(st, n):
    for ins in build_qft(n).instructions:
        if isinstance(ins, Apply):
            apply_gate(st, ins.target, ins.gate)
        else:
            apply_controlled_gate(st, ins.control, ins.target, ins.gate)
    return st


def main():
    out: dict[str, np.ndarray] = {}
    meta: dict[str, str] = {}
    rng = np.random.default_rng(20261017)

    # 1. per-op traces (every target, library + Haar gates, controlled) ------
    for n, n_ops in [(1, 6), (2, 10), (3, 12), (5, 16), (6, 18), (7, 24), (8, 28), (10, 30)]:
        ops, mats, states = trace(n, n_ops, rng)
        out[f"trace{n}_ops"], out[f"trace{n}_mats"], out[f"trace{n}_states"] = ops, mats, states
    # larger registers: final state digest only
    for n, n_ops in [(12, 40), (14, 40)]:
        ops, mats, states = trace(n, n_ops, rng)
        out[f"tracebig{n}_ops"], out[f"tracebig{n}_mats"] = ops, mats
        out[f"tracebig{n}_in"] = states[0]
        meta[f"tracebig{n}_final"] = digest(states[-1])

    # 2. pairsim.random_circuit workloads through run_circuit ----------------
    rc_rng = np.random.default_rng(55)
    for idx in range(6):
        n = int(rc_rng.integers(1, 11))
        circ = random_circuit(n, int(rc_rng.integers(1, 41)), rc_rng)
        st, _ = run_circuit(circ, Precision.SINGLE)
        ops, mats = circuit_arrays(circ)
        out[f"rc{idx}_ops"], out[f"rc{idx}_mats"], out[f"rc{idx}_final"] = ops, mats, st.amps.copy()
        out[f"rc{idx}_n"] = np.array(n)

    # 3. QFT (config 3 shape) on a seeded basis input and an entangled input --
    for n in (6, 10):
        x = int(np.random.default_rng(n).integers(1 << n))
        out[f"qft{n}_basis_x"] = np.array(x)
        out[f"qft{n}_basis"] = run_qft(prep_basis(n, x), n).amps.copy()
        out[f"qft{n}_ent"] = run_qft(prep_entangled(n), n).amps.copy()
    for n in (16, 20):
        x = int(np.random.default_rng(n).integers(1 << n))
        out[f"qft{n}_basis_x"] = np.array(x)
        meta[f"qft{n}_basis"] = digest(run_qft(prep_basis(n, x), n).amps)
        meta[f"qft{n}_ent"] = digest(run_qft(prep_entangled(n), n).amps)

    # 4. config 1: H on every qubit + probabilities ---------------------------
    for n in (12, 20):
        st = new_state(n, Precision.SINGLE)
        for q in range(n):
            apply_gate(st, q, H)
        meta[f"hlayer{n}_amps"] = digest(st.amps)
        meta[f"hlayer{n}_probs"] = digest(probabilities(st))
        if n == 12:
            out["hlayer12_amps"] = st.amps.copy()
            out["hlayer12_probs"] = probabilities(st)

    # 5. sampling and collapse -------------------------------------------------
    def hist_arrays(h):
        keys = np.array(sorted(h.counts), np.int64)
        return keys, np.array([h.counts[k] for k in keys], np.int64)

    samp_states = {
        "rand10": random_state(10, rng).amps.copy(),
        "rand16": random_state(16, rng).amps.copy(),
    }
    sparse = np.zeros(8, np.complex64)
    sparse[[2, 5]] = np.complex64(1 / math.sqrt(2))  # test_measure.py:84-89
    samp_states["sparse3"] = sparse
    st = new_state(14, Precision.SINGLE)
    for q in range(14):
        apply_gate(st, q, H)
    samp_states["hlayer14"] = st.amps.copy()
    # wide dynamic range: probabilities spanning many binades
    w = np.exp(-np.arange(1 << 13) / 300.0) * np.exp(1j * np.arange(1 << 13))
    samp_states["decay13"] = (w / np.linalg.norm(w)).astype(np.complex64)
    for name, amps in samp_states.items():
        n = int(amps.size).bit_length() - 1
        out[f"samp_{name}_amps"] = amps
        for seed in (0, 7, 12345):
            sv = pairsim.StateVector(n, amps.copy())
            keys, counts = hist_arrays(sample(sv, 5000, seed=seed))
            out[f"samp_{name}_s{seed}_keys"], out[f"samp_{name}_s{seed}_counts"] = keys, counts
        coll = []
        for seed in range(20):
            sv = pairsim.StateVector(n, amps.copy())
            m, _ = measure_collapse(sv, seed=seed)
            coll.append(m)
        out[f"samp_{name}_collapse"] = np.array(coll, np.int64)
    # config-1-sized sampling (n=20 H layer), digest of the histogram
    st = new_state(20, Precision.SINGLE)
    for q in range(20):
        apply_gate(st, q, H)
    keys, counts = hist_arrays(sample(st, 100_000, seed=2026))
    meta["samp_hlayer20_s2026"] = digest(np.stack([keys, counts]))

    # 6. Bernstein-Vazirani (pkg/tests/test_acceptance.py:117-128) ----------
    _, hist = run_circuit(build_bernstein_vazirani(14, 101, shots=1000), seed=20260808)
    out["bv14_keys"], out["bv14_counts"] = hist_arrays(hist)

    # 7. Toffoli via pairsim's own gates (6-CNOT decomposition) --------------
    tof_rng = np.random.default_rng(9)
    for (c1, c2, t) in [(0, 1, 2), (4, 0, 2), (1, 3, 0)]:
        st = random_state(5, tof_rng)
        out[f"tof_{c1}{c2}{t}_in"] = st.amps.copy()
        Td = T.dagger()
        seq = [("g", H, t), ("c", X, c2, t), ("g", Td, t), ("c", X, c1, t), ("g", T, t),
               ("c", X, c2, t), ("g", Td, t), ("c", X, c1, t), ("g", T, c2), ("g", T, t),
               ("g", H, t), ("c", X, c1, c2), ("g", T, c1), ("g", Td, c2), ("c", X, c1, c2)]
        for step in seq:
            if step[0] == "g":
                apply_gate(st, step[2], step[1])
            else:
                apply_controlled_gate(st, step[2], step[3], step[1])
        out[f"tof_{c1}{c2}{t}_out"] = st.amps.copy()

    out["meta_keys"] = np.array(list(meta.keys()))
    out["meta_vals"] = np.array(list(meta.values()))
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
