#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-q}
QSB_FUSED_RB=3 timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_${TAG}_rb3.json 2>&1
QSB_FUSED_RB=4 timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_${TAG}_rb4.json 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "Fused or qft or config or smoke or Sweeps or shard" > $OUT/pytest_$TAG.log 2>&1; echo "rc=$?" >> $OUT/pytest_$TAG.log
