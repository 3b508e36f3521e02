"""Per-target sweep time at n=30 for the unfused kernel knobs (QSB_SWEEP_U, QSB_BLOCKS_PER_SM)."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1805_00988_b200 import State
from paper_1805_00988_b200.gates import H
n = 30
st = State(n)
stream = torch.cuda.ExternalStream(st.stream())
targets = [0, 1, 3, 5, 6, 7, 12, 20, 29]
res = {}
for U in sys.argv[1].split(","):
    for B in sys.argv[2].split(","):
        os.environ["QSB_SWEEP_U"], os.environ["QSB_BLOCKS_PER_SM"] = U, B
        row = {}
        for t in targets:
            st.apply_gate(H, t); st.flush()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(5):
                st.apply_gate(H, t)
            b.record(stream); st.flush()
            row[t] = round(a.elapsed_time(b) / 5, 4)
        res[f"U{U}_B{B}"] = row
        print(f"U{U}_B{B}", row, flush=True)
json.dump(res, open("gpurun_out/sweep_tune.json", "w"), indent=1)
