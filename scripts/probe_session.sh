#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python scripts/sample_probe.py > $OUT/sample_probe.log 2>&1
CUDA_VISIBLE_DEVICES=0 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --qubits 24 --no-e2e > $OUT/nccl2_1gpu.log 2>&1; echo "rc=$?" >> $OUT/nccl2_1gpu.log
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"k_fused" -c 2 -o $OUT/prof_qft -f python scripts/profile_qft_pass.py > $OUT/ncu_qft.log 2>&1
