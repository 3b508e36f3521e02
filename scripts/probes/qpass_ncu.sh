mkdir -p gpurun_out
QSB_PROBE_INEXACT=1 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 8 -c 1 -o gpurun_out/ncu_qinx0 -f python scripts/probes/qpass_time.py > gpurun_out/ncu_qinx0.log 2>&1
ncu -i gpurun_out/ncu_qinx0.ncu-rep --page raw --csv > gpurun_out/ncu_qinx0_raw.csv
ncu -i gpurun_out/ncu_qinx0.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_qinx0_sass.csv
