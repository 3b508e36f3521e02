"""H-layer fused passes (light, data-bound) under ring knobs: per-pass time."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
os.environ.setdefault("QSB_FUSED_JIT", "2")
import torch
from paper_1805_00988_b200 import State, build_hadamard_layer, fusion
from paper_1805_00988_b200.circuits import lower_ops
n = 30
st = State(n)
s = torch.cuda.ExternalStream(st.stream())
out = {}
for K in (12, 13):
    passes = fusion.plan(n, lower_ops(build_hadamard_layer(n)), K)
    fusion.run(st, passes); st.flush()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(5):
        fusion.run(st, passes)
    b.record(s); st.flush()
    out[f"K{K}"] = {"passes": len(passes), "ms": a.elapsed_time(b) / 5, "ms_per_pass": a.elapsed_time(b) / 5 / len(passes)}
print(json.dumps(out))
