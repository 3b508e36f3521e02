"""probabilities() of a 30-qubit register into a fresh numpy array (8.6 GB),
host wall clock; run with QSB_PROB_PIECE_LOG / QSB_PROB_NO_HUGE variants."""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
from paper_1805_00988_b200 import State  # noqa: E402

st = State(30)
st.h(0)
st.probabilities(0, 1 << 24)
ts = []
for _ in range(3):
    t0 = time.perf_counter()
    p = st.probabilities()
    ts.append(round((time.perf_counter() - t0) * 1e3, 1))
    del p
print(json.dumps({"ms": ts}))
