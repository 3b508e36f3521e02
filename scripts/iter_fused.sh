#!/bin/bash
# Fused-pass iteration on the GPU box: probe timings, the GPU parity tests,
# and one ncu --set full capture of an H-layer pass and a QFT pass.
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-it}
timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_$TAG.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_$TAG.log
if [ "${2:-}" = "ncu" ]; then
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -c 1 -o $OUT/profh_$TAG -f python scripts/profile_kernels.py --n 30 > $OUT/ncuh_$TAG.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -c 2 -o $OUT/profq_$TAG -f python scripts/profile_qft_pass.py > $OUT/ncuq_$TAG.log 2>&1
fi
echo done
