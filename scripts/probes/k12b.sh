OUT=gpurun_out; : > $OUT/k12b.log
for n in 30 28; do
QSB_FUSED_JIT=2 timeout 300 python - >> $OUT/k12b.log 2>&1 <<PY
import sys, json; sys.path.insert(0, ".")
import torch
from paper_1805_00988_b200 import State, build_hadamard_layer, build_qft, layered_random_circuit, fusion
from paper_1805_00988_b200.circuits import lower_ops
n = $n; st = State(n); s = torch.cuda.ExternalStream(st.stream()); res = {"n": n}
for name, circ in (("hlayer", build_hadamard_layer(n)), ("qft", build_qft(n)), ("layered3", layered_random_circuit(n, 3, seed=32))):
    passes = fusion.plan(n, lower_ops(circ))
    fusion.run(st, passes); st.flush()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(s)
    for _ in range(3): fusion.run(st, passes)
    b.record(s); st.flush()
    res[name] = {"passes": len(passes), "K": len(passes[0].tile), "ms": round(a.elapsed_time(b) / 3, 3)}
print(json.dumps(res))
PY
done
