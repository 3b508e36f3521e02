#!/bin/bash
# One gpurun session: smoke, GPU tests, bench + reference arm, ncu launch list
# of the bench, ncu --set full of the hot kernels (scripts/profile_kernels.py).
# Usage (from repo root, on the GPU box): bash scripts/gpu_session.sh [tag]
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi > $OUT/nvidia_smi_$TAG.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem,power.limit --format=csv >> $OUT/nvidia_smi_$TAG.txt 2>&1
lscpu > $OUT/lscpu_$TAG.txt 2>&1; free -g >> $OUT/lscpu_$TAG.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
timeout 900 python bench.py --steps 10 --warmup 3 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?" >> $OUT/bench_$TAG.err
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-extras > $OUT/ncu_launch_bench_$TAG.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:"k_sweep|k_phase|k_fused|qsb_pass|k_probs|k_chunk_sums|k_trajectories|k_block|k_draws" -c 14 \
    -o $OUT/prof_$TAG -f python scripts/profile_kernels.py --n 30 > $OUT/ncu_full_$TAG.log 2>&1
echo done
