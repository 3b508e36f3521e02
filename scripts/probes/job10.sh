mkdir -p gpurun_out/jitsrc10; rm -f gpurun_out/jitsrc10/*
QSB_FUSED_JIT_DUMP=gpurun_out/jitsrc10 python scripts/qft_passes.py --n 30 --reps 2 > gpurun_out/qp_normal.json 2>&1
QSB_FUSED_DRY=1 python scripts/qft_passes.py --n 30 --reps 2 > gpurun_out/qp_dry1.json 2>&1
QSB_FUSED_DRY=2 python scripts/qft_passes.py --n 30 --reps 2 > gpurun_out/qp_dry2.json 2>&1
QSB_FUSED_DRY=3 python scripts/qft_passes.py --n 30 --reps 2 > gpurun_out/qp_dry3.json 2>&1
cat gpurun_out/qp_*.json
grep -c "while (m)" gpurun_out/jitsrc10/*.cu | head
