"""10^6 exact draws from a 30-qubit register in three states (for ncu)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
from paper_1805_00988_b200 import State
st = State(30)
kind = sys.argv[1] if len(sys.argv) > 1 else "basis"
if kind == "basis":
    st.reset(123456789)
else:
    for q in range(30):
        st.h(q)
    if kind == "generic":
        st.t(3); st.cx(3, 29); st.h(2)
st.sample_outcomes(1000, 1)
st.sample_outcomes(1_000_000, 2)
st.flush()
