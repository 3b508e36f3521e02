"""Per-pass CUDA-event time of the 30-qubit QFT passes (exact; QSB_PROBE_INEXACT=1: exact=False) (compiled
programs), for the ring probes: run under QSB_FUSED_DRY / CTAS_PER_SM knobs."""
import json, os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
os.environ.setdefault("QSB_FUSED_JIT", "2")
import torch
from paper_1805_00988_b200 import State, build_qft, fusion
from paper_1805_00988_b200.circuits import lower_ops
n = 30
st = State(n)
s = torch.cuda.ExternalStream(st.stream())
inexact = os.environ.get("QSB_PROBE_INEXACT") == "1"
passes = fusion.plan(n, lower_ops(build_qft(n)), reorder=inexact)
fusion.run(st, passes, combine=inexact); st.flush()
out = []
for p in passes:
    fusion.run(st, [p], combine=inexact); st.flush()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(5):
        fusion.run(st, [p], combine=inexact)
    b.record(s); st.flush()
    out.append(round(a.elapsed_time(b) / 5, 3))
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("QSB_")}, "ms_per_pass": out,
                  "sum": round(sum(out), 3), "jit": fusion.jit_stats()}))
