"""One fused pass (H on each high tile qubit) over a 32-qubit register for a
compact and a scattered tile: isolates the memory cost of the tile shape."""
import json
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
os.environ.setdefault("QSB_FUSED_JIT", "2")
import torch  # noqa: E402

from paper_1805_00988_b200 import State, fusion  # noqa: E402
from paper_1805_00988_b200.circuits import Apply, Circuit, lower_ops  # noqa: E402
from paper_1805_00988_b200.gates import H  # noqa: E402

n = int(os.environ.get("N", 32))
st = State(n)
s = torch.cuda.ExternalStream(st.stream())
res = {}
for name, high in [("compact", [8, 9, 10, 11, 13, 14]), ("scattered", [16, 20, 25, 26, 27, 29]),
                   ("top", [26, 27, 28, 29, 30, 31]), ("mid", [20, 21, 22, 23, 24, 25])]:
    high = [q for q in high if q < n]
    tile = list(range(6)) + high
    circ = Circuit(n, tuple(Apply(H, q) for q in high))
    arr = fusion.Pass(tile, lower_ops(circ)).op_array()
    st.apply_fused(tile, arr)
    st.flush()
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        st.apply_fused(tile, arr)
        e1.record(s)
        st.flush()
        best = min(best, e0.elapsed_time(e1))
    res[name] = {"ms": round(best, 3), "TBps": round(16 * 2 ** n / best / 1e9, 2)}
print(json.dumps(res))
