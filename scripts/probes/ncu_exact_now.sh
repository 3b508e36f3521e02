export PYTHONPATH=.
timeout 600 ncu --kernel-name regex:qsb_pass --launch-skip 3 --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/qft30_p3 -f python scripts/qft_passes.py --n 30 --reps 0 > /dev/null 2>&1
ncu -i gpurun_out/qft30_p3.ncu-rep --page source --csv --print-source sass > gpurun_out/qft30_p3_sass.csv 2>&1
ncu -i gpurun_out/qft30_p3.ncu-rep --page raw --csv > gpurun_out/qft30_p3_raw.csv 2>&1
python scripts/ncu_brief.py gpurun_out/qft30_p3_raw.csv gpurun_out/qft30_p3_sass.csv > gpurun_out/brief_p3.txt 2>&1
rm -f gpurun_out/*.ncu-rep
cat gpurun_out/brief_p3.txt
