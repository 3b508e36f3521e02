export PYTHONPATH=.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  for part in ${PARTS:-fused sample sample18}; do
    timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_driver.py $part \
      > gpurun_out/sanitize_${tool}_${part}.txt 2>&1
    echo "$tool $part rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|hazard' gpurun_out/sanitize_${tool}_${part}.txt | tail -2 | tr '\n' ' ')"
  done
done
