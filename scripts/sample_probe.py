"""Exact sampling cost at large n (qs_sample: M1..M6 chain)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_1805_00988_b200 import State
res = {}
for n in (24, 28, 30):
    st = State(n)
    for q in range(n):
        st.h(q)
        st.t(q)
    st.sample_outcomes(10, 0)
    for k in (1, 1000, 100000):
        t0 = time.perf_counter(); st.sample_outcomes(k, 1); res[f"n{n}_k{k}_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
    t0 = time.perf_counter(); st.probabilities(); res[f"n{n}_probabilities_ms"] = round((time.perf_counter() - t0) * 1e3, 2)
    st.close()
    print(json.dumps(res), flush=True)
