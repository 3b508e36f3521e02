# Round-2 profile set: launch list of the bench command, ncu --set full per kernel
export PYTHONPATH=.
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r02.csv \
  python bench.py --steps 2 --warmup 1 --no-extras --no-cpu > gpurun_out/launches_bench_r02.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -c 12 -o gpurun_out/kernels_r02 -f \
  python scripts/profile_kernels.py --n 30 > gpurun_out/ncu_kernels_r02.log 2>&1
ncu -i gpurun_out/kernels_r02.ncu-rep --page raw --csv > gpurun_out/kernels_r02_raw.csv 2>&1
python scripts/ncu_brief.py gpurun_out/kernels_r02_raw.csv > gpurun_out/kernels_r02_brief.txt 2>&1
rm -f gpurun_out/*.ncu-rep
python - <<'PY'
import time, ctypes, sys
sys.path.insert(0, '.')
from paper_1805_00988_b200 import _native as N
t0 = time.perf_counter(); a = N.pinned_empty(1 << 30); t1 = time.perf_counter()
print("pinned_empty 8 GiB:", round(t1 - t0, 3), "s")
PY
head -5 gpurun_out/launches_r02.csv; cat gpurun_out/kernels_r02_brief.txt | grep -E "^==|duration|dram"
