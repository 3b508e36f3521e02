QSB_FUSED_JIT=0 python scripts/probes/hpass_time.py
QSB_FUSED_JIT=0 python scripts/probes/qpass_time.py
QSB_FUSED_DRY=1 python scripts/probes/hpass_time.py
python scripts/probes/hpass_time.py
timeout 1500 python -m pytest tests -m gpu -q -x -k 'fused or Fused or jit or Jit or ouble or large or Large or sharded or multidevice' 2>&1 | tail -2
