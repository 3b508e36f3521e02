# sampling chain: timings (both M3 forms), the launch list, parity tests
mkdir -p gpurun_out
python scripts/probes/sample_time.py; python scripts/probes/sample_time.py
QSB_TRAJ_REGS=1 python scripts/probes/sample_time.py
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/samp_generic.csv python scripts/probes/sample_kinds.py generic > /dev/null 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k 'SamplingChain or sample or Sample or measure or Measure or collapse or shard or multidevice or pairsim or double or golden' 2>&1 | tail -3
