import sys; sys.path.insert(0, ".")
from paper_1805_00988_b200 import State, build_qft, execute
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
st = State(n)
for q in range(n): st.h(q)
st.t(3); st.cx(3, 17)
st.sample_outcomes(int(sys.argv[2]) if len(sys.argv) > 2 else 1000000, 2)
st.flush()
