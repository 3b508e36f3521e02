#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/sample_probe.py > $OUT/sample_probe2.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "probabilit or Measurement or shim" > $OUT/pytest_misc.log 2>&1; echo "rc=$?" >> $OUT/pytest_misc.log
timeout 900 python scripts/paper_algorithm2.py --max-qubits 26 --cpu-max-qubits 22 --samples 6 --out $OUT/alg2.csv > $OUT/alg2.txt 2>&1
