# ncu --set full of the sampling chain kernels (10^6 draws, generic 30-qubit state)
mkdir -p gpurun_out
for k in k_chunk_sums_f4 k_trajectories_bulk k_block_walk k_draws; do
ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 \
    -o gpurun_out/ncu_$k -f python scripts/probes/sample_kinds.py generic > gpurun_out/ncu_$k.log 2>&1
ncu -i gpurun_out/ncu_$k.ncu-rep --page raw --csv > gpurun_out/ncu_${k}_raw.csv
ncu -i gpurun_out/ncu_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_${k}_sass.csv
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/samp_generic.csv python scripts/probes/sample_kinds.py generic > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/samp_uniform.csv python scripts/probes/sample_kinds.py uniform > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/samp_basis.csv python scripts/probes/sample_kinds.py basis > /dev/null 2>&1
