"""Per-op cost of the fused tile pass: synthetic op streams on a 30-qubit
register, tile qubits 0..12 (K = 13).  Prints ms per pass for each stream."""
import json, sys, math
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import numpy as np
import torch
from paper_1805_00988_b200 import State, u1
from paper_1805_00988_b200 import _native as N
from paper_1805_00988_b200.gates import m8, H

n = 30
st = State(n)
stream = torch.cuda.ExternalStream(st.stream())
tile = list(range(13))


def ops_array(lst):
    arr = np.zeros(len(lst), dtype=N.OP_DTYPE)
    for i, (kind, t, cm, m) in enumerate(lst):
        arr[i]["kind"], arr[i]["target"], arr[i]["ctrl_mask"], arr[i]["m"] = kind, t, cm, m
    return arr


def timeit(arr, reps=3):
    st.apply_fused(tile, arr); st.flush()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for _ in range(reps):
        st.apply_fused(tile, arr)
    b.record(stream); st.flush()
    return round(a.elapsed_time(b) / reps, 3)


P = N.QS_OP_PHASE; Q = N.QS_OP_PAIR
ph = m8(u1(0.3)); hm = m8(H)
res = {}
res["h_layer13"] = timeit(ops_array([(Q, q, 0, hm) for q in range(13)]))
res["h_lowonly_x13"] = timeit(ops_array([(Q, 1 + (k % 4), 0, hm) for k in range(13)]))  # one LOW stage
res["h_lowonly_x52"] = timeit(ops_array([(Q, 1 + (k % 4), 0, hm) for k in range(52)]))
# phases on lane/warp-only bits of the LOW stage (f >= 4): full 32-amp bodies
res["phase_R0_x100"] = timeit(ops_array([(Q, 1, 0, hm)] + [(P, 9 + (k % 4), 0, ph) for k in range(100)]))
# phases with 3 register bits (2 of 32 amps per thread)
res["phase_R3bits_x100"] = timeit(ops_array([(Q, 1, 0, hm)] + [(P, 2, (1 << 3) | (1 << 4), ph) for k in range(100)]))
# phases whose test fails on an out-of-tile bit for every other tile
res["phase_ext_x100"] = timeit(ops_array([(Q, 1, 0, hm)] + [(P, 20, 0, ph) for k in range(100)]))
# alternating variants (no runs): reg-bit phase patterns cycling
res["phase_alt_x100"] = timeit(ops_array([(Q, 1, 0, hm)] + [(P, 1 + (k % 4), 0, ph) for k in range(100)]))
print(json.dumps(res, indent=1))
