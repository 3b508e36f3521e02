OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_jit.py -q -p no:cacheprovider --durations=5 > $OUT/pytest_jitfile.log 2>&1; tail -12 $OUT/pytest_jitfile.log > $OUT/pytest_jitfile_tail.log
