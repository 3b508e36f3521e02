"""Generate tests/golden/pairsim_golden_double.npz — Precision.DOUBLE (complex128)
outputs of the REFERENCE itself.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden_double.py

Same families as make_golden.py, on complex128 registers: per-op traces
(library + Haar gates, controlled), QFT on basis / entangled inputs, fp64
probabilities, sampling histograms and collapse outcomes, and pairsim's own
6-CNOT Toffoli.  Gate matrices are stored as fp64 (a, b, c, d) entries: for a
complex128 state pairsim's `scalar(x)` rounding (kernel.py:118-119) is exact.
"""

from __future__ import annotations

import math
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent))
from make_golden import REF_SRC, digest, library_gate  # noqa: E402

sys.path.insert(0, str(REF_SRC))
import pairsim  # noqa: E402
from pairsim import (  # noqa: E402
    H,
    T,
    X,
    Apply,
    Precision,
    SerialExecutor,
    apply_controlled_gate,
    apply_gate,
    build_qft,
    measure_collapse,
    new_state,
    probabilities,
    sample,
)

OUT = Path(__file__).resolve().parent / "pairsim_golden_double.npz"
SER = SerialExecutor()
D = Precision.DOUBLE


def m8d(gate) -> np.ndarray:
    vals = [complex(x) for x in (gate.a, gate.b, gate.c, gate.d)]
    return np.array([v for c in vals for v in (c.real, c.imag)], dtype=np.float64)


def random_state(n, rng):
    st = new_state(n, D)
    v = rng.normal(size=st.dim) + 1j * rng.normal(size=st.dim)
    st.amps[:] = v / np.linalg.norm(v)
    return st


def trace(n, n_ops, rng, controlled_fraction=0.4):
    st = random_state(n, rng)
    states = [st.amps.copy()]
    ops, mats = [], []
    for k in range(n_ops):
        gate = library_gate(rng)
        t = k % n if k < n else int(rng.integers(n))
        if n > 1 and rng.random() < controlled_fraction:
            c = int(rng.integers(n - 1))
            c += c >= t
            apply_controlled_gate(st, c, t, gate, SER)
            ops.append((1, c, -1, t))
        else:
            apply_gate(st, t, gate, SER)
            ops.append((0, -1, -1, t))
        mats.append(m8d(gate))
        states.append(st.amps.copy())
    return np.array(ops, np.int32), np.array(mats, np.float64), np.array(states)


def prep_basis(n, x):
    st = new_state(n, D)
    for q in range(n):
        if (x >> q) & 1:
            apply_gate(st, q, X)
    return st


def prep_entangled(n):
    st = new_state(n, D)
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
    rng = np.random.default_rng(20261018)

    for n, n_ops in [(1, 6), (2, 10), (3, 12), (5, 16), (6, 18), (7, 24), (8, 28), (10, 30)]:
        ops, mats, states = trace(n, n_ops, rng)
        out[f"trace{n}_ops"], out[f"trace{n}_mats"], out[f"trace{n}_states"] = ops, mats, states
    for n, n_ops in [(12, 40), (14, 40)]:
        ops, mats, states = trace(n, n_ops, rng)
        out[f"tracebig{n}_ops"], out[f"tracebig{n}_mats"] = ops, mats
        out[f"tracebig{n}_in"] = states[0]
        meta[f"tracebig{n}_final"] = digest(states[-1])

    for n in (6, 10):
        x = int(np.random.default_rng(n).integers(1 << n))
        out[f"qft{n}_basis_x"] = np.array(x)
        out[f"qft{n}_basis"] = run_qft(prep_basis(n, x), n).amps.copy()
        out[f"qft{n}_ent"] = run_qft(prep_entangled(n), n).amps.copy()
    for n in (16,):
        x = int(np.random.default_rng(n).integers(1 << n))
        out[f"qft{n}_basis_x"] = np.array(x)
        meta[f"qft{n}_basis"] = digest(run_qft(prep_basis(n, x), n).amps)
        meta[f"qft{n}_ent"] = digest(run_qft(prep_entangled(n), n).amps)

    st = random_state(10, rng)
    out["probs10_amps"] = st.amps.copy()
    out["probs10"] = probabilities(st)

    def hist_arrays(h):
        keys = np.array(sorted(h.counts), np.int64)
        return keys, np.array([h.counts[k] for k in keys], np.int64)

    w = np.exp(-np.arange(1 << 13) / 300.0) * np.exp(1j * np.arange(1 << 13))
    samp_states = {"rand10": random_state(10, rng).amps.copy(), "decay13": w / np.linalg.norm(w)}
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

    tof_rng = np.random.default_rng(19)
    for (c1, c2, t) in [(0, 1, 2), (4, 0, 2)]:
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

    assert all(v.dtype != np.complex64 for v in out.values())
    out["meta_keys"] = np.array(list(meta.keys()))
    out["meta_vals"] = np.array(list(meta.values()))
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(out)} arrays)")


if __name__ == "__main__":
    main()
