"""Large-register golden digests from the REFERENCE (pairsim), for BASELINE
config 3 (28-qubit QFT vs CPU reference amplitudes) and friends.

    python tests/golden/make_golden_large.py      # ~10 min on 8 cores

Writes tests/golden/pairsim_golden_large.json: SHA-256 of the canonical
complex64 bytes (amplitudes + 0.0f) of each final state, plus the fp64
probabilities digest.  Inputs are rebuilt on the GPU box from the recorded
recipe (basis index x, or the H+T / CX-chain entangled preparation).
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
from make_golden import prep_basis, prep_entangled, run_qft  # noqa: E402
from pairsim import H, apply_gate, new_state, probabilities  # noqa: E402

OUT = Path(__file__).resolve().parent / "pairsim_golden_large.json"


def digest(arr):
    if arr.dtype in (np.complex64, np.float32):
        arr = arr + arr.dtype.type(0)
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


def main(ns=(24, 28)):
    res = json.loads(OUT.read_text()) if OUT.exists() else {}
    for n in ns:
        x = int(np.random.default_rng(n).integers(1 << n))
        t0 = time.time()
        st = run_qft(prep_basis(n, x), n)
        res[f"qft{n}_basis"] = {"x": x, "amps": digest(st.amps), "probs": digest(probabilities(st))}
        del st
        st = run_qft(prep_entangled(n), n)
        res[f"qft{n}_ent"] = {"amps": digest(st.amps), "probs": digest(probabilities(st))}
        del st
        print(f"qft{n}: {time.time() - t0:.0f}s", flush=True)
        OUT.write_text(json.dumps(res, indent=1, sort_keys=True))
    st = new_state(24)
    for q in range(24):
        apply_gate(st, q, H)
    res["hlayer24"] = {"amps": digest(st.amps), "probs": digest(probabilities(st))}
    OUT.write_text(json.dumps(res, indent=1, sort_keys=True))
    print(f"wrote {OUT}")


if __name__ == "__main__":
    main()
