OUT=gpurun_out; : > $OUT/segv2.log
QSB_FUSED_JIT=0 timeout 600 python -m pytest tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider > /dev/null 2>&1; echo "sharded jit0 exit=$?" >> $OUT/segv2.log
QSB_FUSED_JIT=2 timeout 600 python -m pytest tests/test_gpu_sharded.py -m gpu -q -p no:cacheprovider > /dev/null 2>&1; echo "sharded jit2 exit=$?" >> $OUT/segv2.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1805_00988_b200 import State, build_qft, execute
s=State(20); execute(build_qft(20), s); s.flush(); print('queued, exiting')
" >> $OUT/segv2.log 2>&1; echo "inflight exit=$?" >> $OUT/segv2.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1805_00988_b200 import State, build_qft, execute, fusion
s=State(20); execute(build_qft(20), s); s.flush(); fusion.jit_sync(); print('synced, exiting')
" >> $OUT/segv2.log 2>&1; echo "synced exit=$?" >> $OUT/segv2.log
timeout 300 python -c "
import sys; sys.path.insert(0,'.')
from paper_1805_00988_b200 import State, build_qft, execute, fusion
s=State(20); execute(build_qft(20), s); s.flush(); fusion.jit_sync(); s.close(); print('synced+closed, exiting')
" >> $OUT/segv2.log 2>&1; echo "synced_closed exit=$?" >> $OUT/segv2.log
