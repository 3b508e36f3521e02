OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-jit}
QSB_FUSED_JIT=2 timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_$TAG.json 2>&1
QSB_FUSED_JIT=2 timeout 400 ncu --set full --clock-control none --import-source on -k regex:"qsb_pass|k_fused" -c 1 -o $OUT/profq_$TAG -f python scripts/profile_qft_pass.py > $OUT/ncuq_$TAG.log 2>&1
QSB_FUSED_JIT=2 timeout 400 ncu --set full --clock-control none --import-source on -k regex:"qsb_pass|k_fused" -c 1 -o $OUT/profh_$TAG -f python scripts/profile_kernels.py --n 30 > $OUT/ncuh_$TAG.log 2>&1
