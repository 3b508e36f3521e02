"""10^6 exact draws from 30-qubit registers in three states: CUDA-event ms."""
import json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import torch
from paper_1805_00988_b200 import State
st = State(30)
s = torch.cuda.ExternalStream(st.stream())
out = {}
for kind in ("generic", "uniform", "basis"):
    if kind == "basis":
        st.reset(123456789)
    else:
        st.reset(0)
        for q in range(30):
            st.h(q)
        if kind == "generic":
            st.t(3); st.cx(3, 29); st.h(2)
    st.sample_outcomes(1_000_000, 1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s); st.sample_outcomes(1_000_000, 2); b.record(s); st.flush()
    out[kind] = round(a.elapsed_time(b), 3)
print(json.dumps(out))
