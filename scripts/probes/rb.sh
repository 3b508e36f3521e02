OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-rb}
QSB_FUSED_RB=3 timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_${TAG}_rb3.json 2>&1
QSB_FUSED_RB=4 timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_${TAG}_rb4.json 2>&1
