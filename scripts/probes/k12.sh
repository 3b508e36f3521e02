OUT=gpurun_out; : > $OUT/k12.log
for cfg in "13 4 1" "12 4 1" "12 4 2" "12 3 2" "11 3 2" "12 3 1"; do
  set -- $cfg
  echo "K=$1 RB=$2 CTAS=$3" >> $OUT/k12.log
  QSB_FUSED_JIT=2 QSB_FUSED_JIT_RB=$2 QSB_FUSED_CTAS_PER_SM=$3 timeout 300 python scripts/probes/k12_probe.py 30 $1 >> $OUT/k12.log 2>&1
done
