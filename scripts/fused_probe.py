"""Time fused passes (and the TMA ring alone with QSB_FUSED_DRY=1) at n qubits."""
import os, sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
from paper_1805_00988_b200 import State, build_hadamard_layer, build_qft, fusion
from paper_1805_00988_b200.circuits import lower_ops

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
st = State(n)
stream = torch.cuda.ExternalStream(st.stream())
res = {}
for name, circ in (("hlayer", build_hadamard_layer(n)), ("qft", build_qft(n))):
    passes = fusion.plan(n, lower_ops(circ))
    for k, p in enumerate(passes):
        for dry in ("0", "1"):
            os.environ["QSB_FUSED_DRY"] = dry
            st.apply_fused(p.tile, p.op_array()); st.flush()
            a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(3):
                st.apply_fused(p.tile, p.op_array())
            b.record(stream); st.flush()
            res[f"{name}_pass{k}_ops{len(p.ops)}_dry{dry}"] = round(a.elapsed_time(b) / 3, 3)
os.environ["QSB_FUSED_DRY"] = "0"
print(json.dumps(res, indent=1))
