OUT=gpurun_out; : > $OUT/ring.log
for h in 0 1; do
  echo "l2hint=$h" >> $OUT/ring.log
  QSB_FUSED_L2HINT=$h QSB_FUSED_JIT=2 timeout 300 python scripts/fused_probe.py 30 >> $OUT/ring.log 2>&1
  QSB_FUSED_L2HINT=$h QSB_FUSED_JIT=2 timeout 300 python scripts/probes/layered_probe.py 30 >> $OUT/ring.log 2>&1
done
