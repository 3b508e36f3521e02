# Compile-time op program vs interpreter, on the GPU box.
OUT=gpurun_out; mkdir -p $OUT
cd paper_1805_00988_b200/csrc
for name in hlayer qft; do
  rm -f /tmp/dump_$name.txt
  QSB_FUSED_DUMP=/tmp/dump_$name.txt python - <<PY
import sys; sys.path.insert(0, "../..")
from paper_1805_00988_b200 import State, build_hadamard_layer, build_qft, fusion
from paper_1805_00988_b200.circuits import lower_ops
n = 30; st = State(n)
c = build_hadamard_layer(n) if "$name" == "hlayer" else build_qft(n)
p = fusion.plan(n, lower_ops(c)); st.apply_fused(p[0].tile, p[0].op_array()); st.flush()
PY
  python ../../scripts/probes/gen_ops.py /tmp/dump_$name.txt /tmp/gen_$name.inc >> ../../$OUT/gen_exp.log
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -shared -Xcompiler -fPIC -I../../include -I. \
     -DQSB_GEN_OPS='"/tmp/gen_'$name'.inc"' -o /tmp/libgen_$name.so runtime.cu pool.cu gates.cu gates64.cu measure.cu fused.cu 2>&1 | grep -i error >> ../../$OUT/gen_exp.log
done
cd ../..
cat > /tmp/t.py <<'PY'
import sys, json; sys.path.insert(0, ".")
import torch
from paper_1805_00988_b200 import State, build_hadamard_layer, build_qft, fusion
from paper_1805_00988_b200.circuits import lower_ops
n = 30; st = State(n); s = torch.cuda.ExternalStream(st.stream())
name = sys.argv[1]
c = build_hadamard_layer(n) if name == "hlayer" else build_qft(n)
p = fusion.plan(n, lower_ops(c))[0]
arr = p.op_array(); st.apply_fused(p.tile, arr); st.flush()
a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
a.record(s)
for _ in range(5): st.apply_fused(p.tile, arr)
b.record(s); st.flush()
print(name, sys.argv[2], round(a.elapsed_time(b) / 5, 3))
PY
for name in hlayer qft; do
  python /tmp/t.py $name interp >> $OUT/gen_exp.log 2>&1
  QSB_LIB=/tmp/libgen_$name.so python /tmp/t.py $name gen >> $OUT/gen_exp.log 2>&1
done
