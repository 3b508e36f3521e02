# final-build ncu --set full captures: H-layer pass 1, an exact QFT(30) pass, the inexact QFT pass 0
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 8 -c 1 -o gpurun_out/fin_hpass1 -f python scripts/probes/hpass_time.py > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 11 -c 1 -o gpurun_out/fin_qpass -f python scripts/probes/qpass_time.py > /dev/null 2>&1
QSB_PROBE_INEXACT=1 ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 8 -c 1 -o gpurun_out/fin_qinx0 -f python scripts/probes/qpass_time.py > /dev/null 2>&1
for f in fin_hpass1 fin_qpass fin_qinx0; do
  ncu -i gpurun_out/$f.ncu-rep --page raw --csv > gpurun_out/${f}_raw.csv
  ncu -i gpurun_out/$f.ncu-rep --page source --csv --print-source sass > gpurun_out/${f}_sass.csv
done
