# ncu --set full of the sampling chain's M3 (k_trajectories) and M4b
# (k_block_walk), 10^6 draws from a generic 30-qubit state
mkdir -p gpurun_out
for k in ${KERNELS:-k_trajectories k_block_walk}; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/ncu_$k -f python scripts/probes/sample_kinds.py generic > gpurun_out/ncu_$k.log 2>&1
ncu -i gpurun_out/ncu_$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_raw.csv
ncu -i gpurun_out/ncu_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${k}_sass.csv
done
