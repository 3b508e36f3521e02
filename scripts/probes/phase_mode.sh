# QFT(30)/QFT(28) per-pass times for the three diagonal-op code forms (QSB_JIT_PHASE)
export PYTHONPATH=.
for m in 0 1 2; do
  echo "mode $m"
  QSB_JIT_PHASE=$m timeout 300 python scripts/qft_passes.py --n 30
  QSB_JIT_PHASE=$m timeout 300 python scripts/qft_passes.py --n 28
done
