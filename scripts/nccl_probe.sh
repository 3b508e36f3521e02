#!/bin/bash
OUT=gpurun_out; mkdir -p $OUT
NCCL_DEBUG=WARN timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 2 --warmup 1 --qubits 24 > $OUT/nccl2_1gpu.log 2>&1; echo "rc=$?" >> $OUT/nccl2_1gpu.log
