OUT=gpurun_out; : > $OUT/k13rb.log
for cfg in "13 4" "13 3" "12 4" "12 3"; do
  set -- $cfg
  echo "K=$1 RB=$2" >> $OUT/k13rb.log
  QSB_FUSED_JIT=2 QSB_FUSED_JIT_RB=$2 timeout 300 python scripts/probes/k12_probe.py 30 $1 >> $OUT/k13rb.log 2>&1
done
