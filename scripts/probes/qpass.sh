mkdir -p gpurun_out
python scripts/probes/qpass_time.py
QSB_FUSED_DRY=4 python scripts/probes/qpass_time.py
QSB_FUSED_DRY=1 python scripts/probes/qpass_time.py
QSB_PROBE_INEXACT=1 python scripts/probes/qpass_time.py
QSB_FUSED_JIT_RB=4 python scripts/probes/qpass_time.py
QSB_FUSED_JIT_RB=3 python scripts/probes/qpass_time.py
for k in 9 11; do
ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s $k -c 1 -o gpurun_out/ncu_qpass_$k -f python scripts/probes/qpass_time.py > gpurun_out/ncu_qpass_$k.log 2>&1
ncu -i gpurun_out/ncu_qpass_$k.ncu-rep --page raw --csv > gpurun_out/ncu_qpass_${k}_raw.csv
ncu -i gpurun_out/ncu_qpass_$k.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_qpass_${k}_sass.csv
done
