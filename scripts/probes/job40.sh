QSB_JIT_CACHE=0 python scripts/fused_iter.py --big '' 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_jit.py tests/test_gpu_double.py tests/test_gpu_large.py -q -x 2>&1 | tail -3
export PYTHONPATH=.
timeout 600 ncu --kernel-name regex:qsb_pass --launch-skip 5 --launch-count 1 --set full --import-source on \
  --clock-control none -o gpurun_out/c4pass -f python scripts/qft_passes.py --n 28 --reps 0 --circuit layered > /dev/null 2>&1
ncu -i gpurun_out/c4pass.ncu-rep --page source --csv --print-source sass > gpurun_out/c4pass_sass.csv 2>&1
rm -f gpurun_out/*.ncu-rep
python - <<'PY'
import csv, re
rows = list(csv.reader(open('gpurun_out/c4pass_sass.csv')))
hdr = rows[1]
ci = hdr.index('Source'); w = hdr.index('L1 Wavefronts Shared'); wi = hdr.index('L1 Wavefronts Shared Ideal')
tot = [0, 0]
for r in rows[2:]:
    if re.search(r'\b(LDS|STS)', r[ci]):
        tot[0] += int(r[w] or 0); tot[1] += int(r[wi] or 0)
print("LDS/STS wavefronts", tot[0], "ideal", tot[1])
PY
