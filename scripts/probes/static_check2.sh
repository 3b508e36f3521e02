python scripts/probes/hpass_time.py
python scripts/fused_iter.py --big 'QSB_JIT_STATIC_STAGES=1' > gpurun_out/static_iter2.jsonl 2>&1
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:qsb_pass -s 8 -c 1 -o gpurun_out/ncu_hpass1 -f python scripts/probes/hpass_time.py > gpurun_out/ncu_hpass1.log 2>&1
ncu -i gpurun_out/ncu_hpass1.ncu-rep --page raw --csv > gpurun_out/ncu_hpass1_raw.csv
ncu -i gpurun_out/ncu_hpass1.ncu-rep --page source --csv --print-source sass > gpurun_out/ncu_hpass1_sass.csv
timeout 1500 python -m pytest tests -m gpu -q -x -k 'fused or Fused or jit or Jit' 2>&1 | tail -3
