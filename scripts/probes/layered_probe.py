"""Time the fused passes of the config-4 workload shape (layered H/T/CX) at n qubits,
compiled (QSB_FUSED_JIT=2) and data-only (QSB_FUSED_DRY=1)."""
import os, sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import torch
from paper_1805_00988_b200 import State, layered_random_circuit, fusion
from paper_1805_00988_b200.circuits import lower_ops
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
st = State(n); s = torch.cuda.ExternalStream(st.stream())
passes = fusion.plan(n, lower_ops(layered_random_circuit(n, 3, seed=32)))
res = {"passes": len(passes)}
for k, p in enumerate(passes[:8]):
    arr = p.op_array()
    kinds = {}
    for (kind, t, cm, m) in p.ops:
        key = ("phase" if kind == 1 else ("cx" if cm else "1q"))
        kinds[key] = kinds.get(key, 0) + 1
    for dry in ("0", "1"):
        os.environ["QSB_FUSED_DRY"] = dry
        st.apply_fused(p.tile, arr); st.flush()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(3): st.apply_fused(p.tile, arr)
        b.record(s); st.flush()
        res[f"pass{k}_{kinds}_dry{dry}"] = round(a.elapsed_time(b) / 3, 3)
print(json.dumps(res, indent=1))
