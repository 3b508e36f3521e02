"""Circuit workflow variants (n = 30 H layer + 1000 shots): per-step CUDA-event ms."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import torch
from paper_1805_00988_b200 import State, build_hadamard_layer, fusion
from paper_1805_00988_b200.circuits import lower_ops
n = 30
st = State(n)
s = torch.cuda.ExternalStream(st.stream())
passes = fusion.plan(n, lower_ops(build_hadamard_layer(n)))
def plain(k):
    st.reset(0); fusion.run(st, passes); return st.sample_outcomes(1000, k)
def folded(k):
    fusion.run(st, passes, from_basis=0); return st.sample_outcomes(1000, k)
def folded_sums(k):
    st.sample_prepare(1000); r = fusion.run(st, passes, from_basis=0, chunk_sums=True)
    return st.sample_outcomes(1000, k, sums_ready=r)
def passes_only_sums(k):
    st.sample_prepare(1000); fusion.run(st, passes, from_basis=0, chunk_sums=True)
def passes_only(k):
    fusion.run(st, passes, from_basis=0)
out = {}
for name, f in (("plain", plain), ("folded", folded), ("folded_sums", folded_sums), ("passes_only", passes_only),
                ("passes_only_sums", passes_only_sums), ("plain2", plain), ("folded_sums2", folded_sums)):
    for k in range(2):
        f(k)
    fusion.jit_sync(); st.flush()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); a.record(s)
    for k in range(10):
        f(k)
    b.record(s); st.flush()
    out[name] = {"event_ms": round(a.elapsed_time(b) / 10, 3), "wall_ms": round((time.perf_counter() - t0) * 100, 3)}
print(json.dumps(out))
