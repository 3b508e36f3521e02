for d in 0 1 4; do QSB_FUSED_DRY=$d python scripts/qft_passes.py --n 30 --reps 2 > gpurun_out/qp12_dry$d.json 2>&1; done
cat gpurun_out/qp12_*.json
timeout 900 python -m pytest tests/test_gpu_fault.py -q 2>&1 | tail -4
