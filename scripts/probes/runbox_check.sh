# fused passes with run-merged TMA boxes vs one-bit box dims: timing + parity
mkdir -p gpurun_out
python scripts/fused_iter.py --big 'QSB_FUSED_RUN_BOXES=0' 'QSB_FUSED_RUN_BOXES=1' > gpurun_out/runbox_iter.jsonl 2>&1
python scripts/probes/ring_iter.py > gpurun_out/runbox_ring1.json 2>&1
QSB_FUSED_RUN_BOXES=0 python scripts/probes/ring_iter.py > gpurun_out/runbox_ring0.json 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x -k 'fused or Fused or jit or Jit or large or Large or sharded or multidevice or double' 2>&1 | tail -3
