"""Per-pass CUDA-event time of the four 30-qubit H-layer passes (compiled
programs), for the ring probes: run under QSB_FUSED_DRY / CTAS_PER_SM knobs."""
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
passes = fusion.plan(n, lower_ops(build_hadamard_layer(n)), 12)
fusion.run(st, passes); st.flush()
out = []
for p in passes:
    fusion.run(st, [p]); st.flush()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(5):
        fusion.run(st, [p])
    b.record(s); st.flush()
    out.append(round(a.elapsed_time(b) / 5, 3))
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("QSB_")}, "ms_per_pass": out,
                  "sum": round(sum(out), 3), "jit": fusion.jit_stats()}))
