"""FP32-pipe efficiency of compiled diagonal ops: one pass of M u1 gates on a
single qubit q of an n-qubit register (q = 1: a register bit of the LOW
stage -> unconditional straight-line phase_ct; q = 6: a lane bit -> a
divergent conditional body; q = 20: a tile-uniform test).  Floor = M * 2^(n-1)
amplitudes * 4 FP32 lane-ops / (148 SMs * 128 lanes * clock)."""
import json
import math
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
os.environ.setdefault("QSB_FUSED_JIT", "2")
import torch  # noqa: E402

from paper_1805_00988_b200 import State, u1  # noqa: E402
from paper_1805_00988_b200.circuits import Apply, Circuit, lower_ops  # noqa: E402
from paper_1805_00988_b200 import fusion  # noqa: E402

n = 28
st = State(n)
s = torch.cuda.ExternalStream(st.stream())
res = {}
cases = [(1, None), (6, None), (20, None)]
if len(sys.argv) > 1:
    cases = [(int(x), None) for x in sys.argv[1].split(",")]
for q, tile in cases:
    for M in (150,):
        circ = Circuit(n, tuple(Apply(u1(0.1 + 1e-3 * i), q) for i in range(M)))
        tq = tile or list(range(13))
        passes = [fusion.Pass(tq, lower_ops(circ))]
        arr = passes[0].op_array()
        st.apply_fused(tq, arr)
        st.flush()
        best = 1e9
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            st.apply_fused(tq, arr)
            e1.record(s)
            st.flush()
            best = min(best, e0.elapsed_time(e1))
        floor = M * 2 ** (n - 1) * 4 / (148 * 128 * 1.965e9) * 1e3
        res[f"q{q}_M{M}"] = {"ms": round(best, 3), "fp32_floor_ms": round(floor, 3), "frac": round(floor / best, 3)}
print(json.dumps(res))
