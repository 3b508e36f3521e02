"""Launch the first fused pass of QFT(30) (compiled, default tile choice) and
one pass of the layered config-4 circuit, for ncu."""
import os
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1805_00988_b200 import State, build_qft, layered_random_circuit, fusion  # noqa: E402
from paper_1805_00988_b200.circuits import lower_ops  # noqa: E402
os.environ.setdefault("QSB_FUSED_JIT", "2")
n = 30
st = State(n)
p = fusion.plan(n, lower_ops(build_qft(n)))
st.apply_fused(p[0].tile, p[0].op_array())
q = fusion.plan(n, lower_ops(layered_random_circuit(n, 4, seed=32)))
st.apply_fused(q[1].tile, q[1].op_array())
st.flush()
print("ops", len(p[0].ops), len(q[1].ops), "K", len(p[0].tile), len(q[1].tile))
