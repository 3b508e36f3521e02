"""probabilities() of a 30-qubit register into a fresh numpy array: host ms."""
import json, os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
from paper_1805_00988_b200 import State
st = State(30)
for q in range(30):
    st.h(q)
st.flush()
best = 1e9
for _ in range(3):
    t0 = time.perf_counter(); p = st.probabilities(); dt = time.perf_counter() - t0
    best = min(best, dt); del p
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("QSB_PROB")}, "ms": round(best * 1e3, 1)}))
