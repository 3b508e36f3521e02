"""QFT(30) exact fused at K = 12 / 13 and CTAs per SM settings (compiled)."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
os.environ.setdefault("QSB_FUSED_JIT", "2")
import torch
from paper_1805_00988_b200 import State, build_qft, fusion
from paper_1805_00988_b200.circuits import lower_ops
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
st = State(n)
s = torch.cuda.ExternalStream(st.stream())
out = {}
for K in (12, 13):
    passes = fusion.plan(n, lower_ops(build_qft(n)), K)
    fusion.run(st, passes); st.flush()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(3):
        fusion.run(st, passes)
    b.record(s); st.flush()
    out[f"K{K}"] = {"passes": len(passes), "ms": a.elapsed_time(b) / 3}
print(json.dumps(out))
