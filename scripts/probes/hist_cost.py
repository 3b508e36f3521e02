"""pairsim.sample (histogram) cost split: device outcomes vs host np.unique + dict."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import numpy as np
from paper_1805_00988_b200 import pairsim as ps
from paper_1805_00988_b200 import build_hadamard_layer, build_bernstein_vazirani
out = {}
for name, circ in (("hlayer26", build_hadamard_layer(26)), ("bv26", build_bernstein_vazirani(26, 12345, shots=1))):
    from paper_1805_00988_b200.circuits import Circuit
    c = Circuit(circ.num_qubits, tuple(i for i in circ.instructions if type(i).__name__ != "SampleMeasure"))
    st, _ = ps.run_circuit(c)
    ps.sample(st, 1000, 1)
    t0 = time.perf_counter(); o = st.device_state.sample_outcomes(10**6, 2); t1 = time.perf_counter()
    k, n = np.unique(o, return_counts=True); t2 = time.perf_counter()
    d = {int(a): int(b) for a, b in zip(k, n)}; t3 = time.perf_counter()
    h = ps.sample(st, 10**6, 2); t4 = time.perf_counter()
    out[name] = {"outcomes_ms": (t1 - t0) * 1e3, "unique_ms": (t2 - t1) * 1e3, "dict_ms": (t3 - t2) * 1e3,
                 "pairsim_sample_ms": (t4 - t3) * 1e3, "distinct": len(d)}
print(json.dumps(out))
