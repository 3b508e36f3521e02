export PYTHONPATH=.
mkdir -p gpurun_out/jitsrc_inx; rm -f gpurun_out/jitsrc_inx/*
QSB_FUSED_JIT_DUMP=gpurun_out/jitsrc_inx python scripts/qft_passes.py --n 30 --reps 2 --inexact > gpurun_out/qp_inexact.json 2>&1
timeout 600 ncu --kernel-name regex:qsb_pass --launch-skip 2 --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/qft30_inx -f python scripts/qft_passes.py --n 30 --reps 0 --inexact > gpurun_out/ncu_inx.log 2>&1
ncu -i gpurun_out/qft30_inx.ncu-rep --page source --csv --print-source sass > gpurun_out/qft30_inx_sass.csv 2>&1
ncu -i gpurun_out/qft30_inx.ncu-rep --page raw --csv > gpurun_out/qft30_inx_raw.csv 2>&1
python scripts/ncu_brief.py gpurun_out/qft30_inx_raw.csv gpurun_out/qft30_inx_sass.csv > gpurun_out/brief_inx.txt 2>&1
rm -f gpurun_out/*.ncu-rep
cat gpurun_out/qp_inexact.json gpurun_out/brief_inx.txt
