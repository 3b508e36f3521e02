"""Fused-pass perf iteration: for each knob setting (environment variables,
one subprocess each) time the compiled fused circuits of the bench extras and
check them bit-for-bit against the unfused sweeps at a smaller width.

    python scripts/fused_iter.py [--big] 'QSB_JIT_SEL=0' 'QSB_JIT_SEL=1' ...

Prints one JSON line per setting.  (Builder tooling, not product.)
"""
from __future__ import annotations

import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CHILD = r'''
import json, os, sys, time
sys.path.insert(0, {root!r})
import numpy as np, torch
from paper_1805_00988_b200 import State, build_qft, build_hadamard_layer, layered_random_circuit, fusion, execute
from paper_1805_00988_b200.circuits import lower_ops
out = {{}}
def timed(n, circ, reps=3, exact=True):
    st = State(n)
    s = torch.cuda.ExternalStream(st.stream())
    passes = fusion.plan(n, lower_ops(circ), reorder=not exact)
    t0 = time.perf_counter()
    fusion.run(st, passes, combine=not exact); st.flush()
    cold = time.perf_counter() - t0
    fusion.jit_sync()
    fusion.run(st, passes, combine=not exact); st.flush()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(reps):
        fusion.run(st, passes, combine=not exact)
    b.record(s); st.flush()
    st.close()
    return {{"ms": a.elapsed_time(b) / reps, "passes": len(passes), "cold_ms": cold * 1e3}}
def exact(n, circ):
    a, b = State(n), State(n)
    execute(circ, a, fuse=True); fusion.jit_sync(); a.reset(0); execute(circ, a, fuse=True)
    execute(circ, b, fuse=False)
    x, y = a.amplitudes(), b.amplitudes()
    a.close(); b.close()
    return bool(np.all(x == y))
out["exact_qft22"] = exact(22, build_qft(22))
out["exact_layered22"] = exact(22, layered_random_circuit(22, 12, seed=5))
out["qft28"] = timed(28, build_qft(28))
out["qft30"] = timed(30, build_qft(30))
out["hlayer30"] = timed(30, build_hadamard_layer(30))
out["qft28_inexact"] = timed(28, build_qft(28), exact=False)
out["qft30_inexact"] = timed(30, build_qft(30), exact=False)
if {big!r}:
    out["config4_32"] = timed(32, layered_random_circuit(32, 20, seed=32), reps=1)
    out["config4_32_inexact"] = timed(32, layered_random_circuit(32, 20, seed=32), reps=1, exact=False)
print(json.dumps(out))
'''


def main():
    big = "--big" in sys.argv
    settings = [a for a in sys.argv[1:] if not a.startswith("--")] or [""]
    for setting in settings:
        env = dict(os.environ)
        for kv in setting.split():
            k, v = kv.split("=", 1)
            env[k] = v
        r = subprocess.run([sys.executable, "-c", CHILD.format(root=str(ROOT), big=big)], env=env,
                           capture_output=True, text=True, timeout=900)
        line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else ""
        try:
            res = json.loads(line)
        except json.JSONDecodeError:
            res = {"error": (r.stderr or r.stdout)[-1500:]}
        print(json.dumps({"setting": setting, **res}), flush=True)


if __name__ == "__main__":
    main()
