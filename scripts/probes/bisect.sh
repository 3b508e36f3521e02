OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/bisect.log 2>&1; tail -3 $OUT/bisect.log > $OUT/bisect_tail.log
timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_f3.json 2>&1
