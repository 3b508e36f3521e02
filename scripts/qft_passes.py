"""Per-pass device time of the fused QFT(n) (compiled programs), for the
planner / program work.  With QSB_FUSED_DUMP=<file> the stage plans are
appended to <file>.  Run under ncu to get per-pass instruction counts.

    python scripts/qft_passes.py [--n 30] [--reps 3] [--k K]
"""
import argparse
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
os.environ.setdefault("QSB_FUSED_JIT", "2")

import torch  # noqa: E402

from paper_1805_00988_b200 import State, build_qft, fusion  # noqa: E402
from paper_1805_00988_b200.circuits import lower_ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--k", type=int, default=None)
ap.add_argument("--circuit", default="qft")
ap.add_argument("--inexact", action="store_true", help="reorder planner + combined diagonal runs")
a = ap.parse_args()
n = a.n
st = State(n)
if a.circuit == "qft":
    circ = build_qft(n)
else:
    from paper_1805_00988_b200 import layered_random_circuit
    circ = layered_random_circuit(n, 20, seed=32)
passes = fusion.plan(n, lower_ops(circ), a.k, reorder=a.inexact)
s = torch.cuda.ExternalStream(st.stream())
out = []
dump = os.environ.pop("QSB_FUSED_DUMP", None)
for i, p in enumerate(passes):
    arr = p.op_array()
    if dump:
        os.environ["QSB_FUSED_DUMP"] = dump
    st.apply_fused(p.tile, arr, combine=a.inexact)  # compile + warm (+ dump this pass's plan once)
    st.flush()
    os.environ.pop("QSB_FUSED_DUMP", None)
    ts = []
    for _ in range(a.reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        st.apply_fused(p.tile, arr, combine=a.inexact)
        e1.record(s)
        st.flush()
        ts.append(e0.elapsed_time(e1))
    nph = sum(1 for op in p.ops if op[0] == 1)
    out.append({"pass": i, "tile": list(p.tile), "ops": len(p.ops), "phase_ops": nph, "ms": min(ts) if ts else None})
print(json.dumps({"n": n, "total_ms": sum(o["ms"] or 0 for o in out), "passes": out}))
