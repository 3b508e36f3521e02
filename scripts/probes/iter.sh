# tests + fused probe (+ optional ncu of the fused passes)
OUT=gpurun_out; mkdir -p $OUT; TAG=${1:-it}
timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider > $OUT/pytest_$TAG.log 2>&1; tail -3 $OUT/pytest_$TAG.log > $OUT/pytest_tail_$TAG.log
timeout 300 python scripts/fused_probe.py 30 > $OUT/probe_$TAG.json 2>&1
if [ "${2:-}" = "ncu" ]; then bash scripts/probes/ncu_fused.sh $TAG; fi
