# full ncu capture of QFT(30) fused pass 1 (compiled) + generated sources and stage plans
export PYTHONPATH=.
mkdir -p gpurun_out/jitsrc; rm -f gpurun_out/jitsrc/* gpurun_out/plan_qft30.txt
QSB_FUSED_JIT_DUMP=gpurun_out/jitsrc QSB_FUSED_DUMP=gpurun_out/plan_qft30.txt timeout 300 python scripts/qft_passes.py --n 30 --reps 2 > gpurun_out/qft_passes_${1:-a}.json 2>&1
timeout 600 ncu --kernel-name regex:qsb_pass --launch-skip 1 --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/qft30_pass1_${1:-a} -f python scripts/qft_passes.py --n 30 --reps 0 > gpurun_out/ncu_qft_pass_${1:-a}.log 2>&1
ncu -i gpurun_out/qft30_pass1_${1:-a}.ncu-rep --page source --csv --print-source sass > gpurun_out/qft30_pass1_${1:-a}_sass.csv 2>&1
ncu -i gpurun_out/qft30_pass1_${1:-a}.ncu-rep --page raw --csv > gpurun_out/qft30_pass1_${1:-a}_raw.csv 2>&1
ls -la gpurun_out/ | head -30
