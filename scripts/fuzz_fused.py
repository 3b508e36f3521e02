"""Randomised parity sweep of the fused passes (builder tooling): random
circuits — library / Haar / u1 gates, controlled and doubly-controlled, all
gate classes — over random register sizes and tile widths, run as compiled
pass programs (and the interpreter kernel for a share of them) and compared
bit for bit with the unfused sweeps on the same register; every third case
also as a measured circuit from a basis state (the folded reset and the
last pass's row sums) against reset + sweeps + the plain sampler (values
and draws).  Exits non-zero on
the first mismatch and prints the failing case.

    python scripts/fuzz_fused.py [cases] [seed]
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("QSB_FUSED_JIT", "2")

import numpy as np  # noqa: E402

from paper_1805_00988_b200 import State, fusion, random_circuit  # noqa: E402
from paper_1805_00988_b200.circuits import (  # noqa: E402
    Circuit, ControlledControlledApply, SampleMeasure, execute, lower_ops)
from paper_1805_00988_b200.gates import FIXED_GATES, random_unitary_gate  # noqa: E402


def with_ccx(circ: Circuit, rng, count: int) -> Circuit:
    ins = list(circ.instructions)
    n = circ.num_qubits
    for _ in range(count):
        c1, c2, t = rng.choice(n, 3, replace=False)
        g = FIXED_GATES["x"] if rng.random() < 0.5 else random_unitary_gate(rng)
        ins.insert(int(rng.integers(0, len(ins) + 1)), ControlledControlledApply(g, int(c1), int(c2), int(t)))
    return Circuit(n, tuple(ins))


def main() -> int:
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 120
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 2026
    rng = np.random.default_rng(seed)
    t0 = time.time()
    stats = {"cases": 0, "ops": 0, "passes": 0}
    for case in range(cases):
        n = int(rng.integers(10, 21))
        depth = int(rng.integers(2, 40))
        K = int(rng.integers(10, min(13, n) + 1))
        circ = with_ccx(random_circuit(n, depth, rng), rng, int(rng.integers(0, 6)))
        a0 = (rng.normal(size=1 << n) + 1j * rng.normal(size=1 << n)).astype(np.complex64)
        ref = State(n)
        ref.set_amplitudes(a0)
        execute(circ, ref, fuse=False)
        want = ref.amplitudes()
        ref.close()
        passes = fusion.plan(n, lower_ops(circ), K)
        for jit in ("2",) + (("0",) if case % 4 == 0 else ()):  # compiled; every 4th case also interpreted
            os.environ["QSB_FUSED_JIT"] = jit  # read per call by the library
            st = State(n)
            st.set_amplitudes(a0)
            fusion.run(st, passes)
            got = st.amplitudes()
            st.close()
            if got.tobytes() != want.tobytes():
                bad = int(np.flatnonzero(got.view(np.uint64) != want.view(np.uint64))[0])
                print(json.dumps({"mismatch": True, "case": case, "n": n, "K": K, "depth": depth,
                                  "jit": os.environ.get("QSB_FUSED_JIT"), "first_index": bad,
                                  "got": str(got[bad]), "want": str(want[bad])}))
                return 1
        os.environ["QSB_FUSED_JIT"] = "2"
        if case % 3 == 0:  # the measured-circuit path: folded reset + row sums left by the last pass
            b = int(rng.integers(0, 1 << n))
            shots = int(rng.integers(1, 3000))
            ref = State(n)
            ref.reset(b)
            execute(circ, ref, fuse=False)
            want_amp = ref.amplitudes()
            want_out = ref.sample_outcomes(shots, case)
            ref.close()
            st = State(n)
            st.set_amplitudes(a0)  # stale contents
            got_out = execute(Circuit(n, circ.instructions + (SampleMeasure(shots),)), st, seed=case,
                              tile_qubits=K, initial_basis=b)
            got_amp = st.amplitudes()
            st.close()
            # values, not bytes: from a basis state the register holds exact
            # zeros, and fused diagonal ops may flip their sign (the documented
            # freedom: 1*x + 0*y adds +-0, same as the sweeps up to the sign of 0)
            if not np.array_equal(got_amp, want_amp) or not np.array_equal(got_out, want_out):
                print(json.dumps({"mismatch": True, "case": case, "n": n, "K": K, "mode": "measured", "basis": b}))
                return 1
            stats["measured"] = stats.get("measured", 0) + 1
        stats["cases"] += 1
        stats["ops"] += len(circ.instructions)
        stats["passes"] += len(passes)
    print(json.dumps({"mismatch": False, **stats, "jit": fusion.jit_stats(), "seconds": round(time.time() - t0, 1)}))
    return 0


if __name__ == "__main__":
    sys.exit(main())
