#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-q}
timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_$TAG.json 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "Fused or qft or config or smoke or Sweeps" > $OUT/pytest_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_$TAG.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -c 1 -o $OUT/prof_$TAG -f python scripts/profile_kernels.py --n 30 > $OUT/ncu_$TAG.log 2>&1
