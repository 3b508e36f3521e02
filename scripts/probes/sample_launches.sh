mkdir -p gpurun_out
for k in generic uniform basis; do
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/samp_$k.csv python scripts/probes/sample_kinds.py $k > /dev/null 2>&1
done
python scripts/ncu_brief.py --help >/dev/null 2>&1; true
