# dump the generated pass programs of the H layer / QFT(30) / config 4 (JIT cache off)
mkdir -p gpurun_out/jit_dump
export QSB_JIT_DUMP=gpurun_out/jit_dump QSB_JIT_CACHE=0
python scripts/probes/hpass_time.py
