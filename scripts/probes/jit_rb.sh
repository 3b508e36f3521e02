OUT=gpurun_out; mkdir -p $OUT
for rb in 4 5; do
QSB_FUSED_JIT=2 QSB_FUSED_JIT_RB=$rb QSB_FUSED_JIT_VERBOSE=1 timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_jitrb$rb.json 2>&1
done
QSB_FUSED_JIT=2 QSB_FUSED_JIT_RB=5 QSB_FUSED_JIT_VERBOSE=1 timeout 600 python -m pytest tests/test_gpu_jit.py -q -p no:cacheprovider > $OUT/pytest_jitrb5.log 2>&1; tail -3 $OUT/pytest_jitrb5.log > $OUT/pytest_jitrb5_tail.log
timeout 600 python -m pytest tests/test_gpu_jit.py -q -p no:cacheprovider > $OUT/pytest_jitrb4.log 2>&1; tail -3 $OUT/pytest_jitrb4.log > $OUT/pytest_jitrb4_tail.log
