./scripts/probes/cmul_rate > gpurun_out/cmul_rate.txt 2>&1
python scripts/fused_iter.py 'QSB_JIT_PLANAR=0' 'QSB_JIT_PLANAR=2' 'QSB_JIT_PLANAR=2 QSB_JIT_SEL=0' > gpurun_out/iter3.jsonl 2>&1
bash scripts/probes/ncu_qft_now.sh p2 > /dev/null 2>&1
python scripts/ncu_brief.py gpurun_out/qft30_pass1_p2_raw.csv gpurun_out/qft30_pass1_p2_sass.csv > gpurun_out/brief_p2.txt 2>&1
rm -f gpurun_out/*.ncu-rep
cat gpurun_out/cmul_rate.txt gpurun_out/iter3.jsonl gpurun_out/brief_p2.txt
