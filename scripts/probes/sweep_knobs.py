"""Headline sweep (H on every target, n = 30) under QSB_SWEEP_U / QSB_BLOCKS_PER_SM."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import torch
from paper_1805_00988_b200 import State
st = State(30)
s = torch.cuda.ExternalStream(st.stream())
for q in range(30):
    st.h(q)
st.flush()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(3):
    for q in range(30):
        st.h(q)
b.record(s); st.flush()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("QSB_")},
                  "ms_per_sweep": round(a.elapsed_time(b) / 90, 4)}))
