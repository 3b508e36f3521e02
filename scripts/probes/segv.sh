OUT=gpurun_out
# which test file's process segfaults at exit?
for f in tests/test_gpu_jit.py tests/test_gpu_parity.py tests/test_gpu_double.py tests/test_gpu_sharded.py tests/test_pairsim_shim.py tests/test_qc.py; do
  timeout 600 python -X faulthandler -m pytest $f -m gpu -q -p no:cacheprovider > $OUT/segv_$(basename $f).log 2>&1
  echo "$f exit=$?" >> $OUT/segv.log
done
