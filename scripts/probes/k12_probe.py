"""Fused pass timings for H layer / QFT / layered circuits at n qubits with a
given tile size (argv[2]); run under different QSB_FUSED_* settings."""
import os, sys, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import torch
from paper_1805_00988_b200 import State, build_hadamard_layer, build_qft, layered_random_circuit, fusion
from paper_1805_00988_b200.circuits import lower_ops
n = int(sys.argv[1]); K = int(sys.argv[2])
st = State(n); s = torch.cuda.ExternalStream(st.stream())
res = {}
for name, circ in (("hlayer", build_hadamard_layer(n)), ("qft", build_qft(n)), ("layered3", layered_random_circuit(n, 3, seed=32))):
    passes = fusion.plan(n, lower_ops(circ), K)
    fusion.run(st, passes); fusion.run(st, passes); st.flush()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(3): fusion.run(st, passes)
    b.record(s); st.flush()
    res[name] = {"passes": len(passes), "ms": round(a.elapsed_time(b) / 3, 3)}
print(json.dumps({"K": K, **res}))
