timeout 900 python -m pytest tests -m gpu -x -q -k 'multidevice or sharded_mp or sharded' 2>&1 | tail -15 > gpurun_out/gputest_r02c.txt
bash scripts/probes/ncu_qft_now.sh inter
QSB_JIT_PLANAR=1 bash scripts/probes/ncu_qft_now.sh planar
python scripts/ncu_brief.py gpurun_out/qft30_pass1_inter_raw.csv gpurun_out/qft30_pass1_inter_sass.csv > gpurun_out/brief_inter.txt 2>&1
python scripts/ncu_brief.py gpurun_out/qft30_pass1_planar_raw.csv gpurun_out/qft30_pass1_planar_sass.csv > gpurun_out/brief_planar.txt 2>&1
rm -f gpurun_out/*.ncu-rep
