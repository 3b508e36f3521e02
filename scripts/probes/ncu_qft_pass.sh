# full ncu capture (with SASS-level warp-state samples) of QFT(30) fused pass 1 (compiled)
export PYTHONPATH=.
timeout 600 ncu --kernel-name regex:qsb_pass --launch-skip 1 --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/qft30_pass1 -f python scripts/qft_passes.py --n 30 --reps 0 > gpurun_out/ncu_qft_pass.log 2>&1
ncu -i gpurun_out/qft30_pass1.ncu-rep --page source --csv --print-source sass > gpurun_out/qft30_pass1_sass.csv 2>&1
ls -la gpurun_out/qft30_pass1*
