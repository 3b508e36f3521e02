OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-nf}
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -c 1 -o $OUT/profh_$TAG -f python scripts/profile_kernels.py --n 30 > $OUT/ncuh_$TAG.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -c 1 -o $OUT/profq_$TAG -f python scripts/profile_qft_pass.py > $OUT/ncuq_$TAG.log 2>&1
