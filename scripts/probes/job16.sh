mkdir -p gpurun_out/jitsrc16; rm -f gpurun_out/jitsrc16/*
QSB_FUSED_JIT_DUMP=gpurun_out/jitsrc16 QSB_JIT_TILE_LOOP=3 python scripts/qft_passes.py --n 30 --reps 2 > gpurun_out/qp16_loop.json 2>&1
QSB_JIT_TILE_LOOP=0 python scripts/qft_passes.py --n 30 --reps 2 > gpurun_out/qp16_noloop.json 2>&1
cat gpurun_out/qp16_loop.json gpurun_out/qp16_noloop.json
grep -c "while (m)" gpurun_out/jitsrc16/*.cu
timeout 600 python -m pytest tests -m gpu -q -x -k "shard or multidevice" 2>&1 | tail -3
bash scripts/sanitize.sh
