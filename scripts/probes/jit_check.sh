OUT=gpurun_out; mkdir -p $OUT
QSB_FUSED_JIT=2 QSB_FUSED_JIT_VERBOSE=1 timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "Fused or fused or qft or config or smoke or Config" > $OUT/pytest_jit.log 2>&1; tail -5 $OUT/pytest_jit.log > $OUT/pytest_jit_tail.log
QSB_FUSED_JIT=2 QSB_FUSED_JIT_VERBOSE=1 timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_jit.json 2>&1
QSB_FUSED_JIT=2 timeout 300 python scripts/probes/op_cost.py > $OUT/op_cost_jit.json 2>&1
