mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_full.log 2>&1; tail -3 gpurun_out/pytest_full.log
timeout 1200 python bench.py > gpurun_out/bench_r02s.json 2> gpurun_out/bench_r02s.err; tail -c 300 gpurun_out/bench_r02s.err
python -c 'import __graft_entry__ as g; g.smoke(); print("smoke ok")'
