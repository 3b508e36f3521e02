python scripts/probes/hpass_time.py
python scripts/fused_iter.py --big 'QSB_JIT_STATIC_STAGES=1' > gpurun_out/static_iter3.jsonl 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k 'fused or Fused or jit or Jit or large or Large' 2>&1 | tail -3
