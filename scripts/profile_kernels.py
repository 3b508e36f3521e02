"""Launch exactly the kernels we want ncu to capture (run under ncu on the GPU box).

    python scripts/profile_kernels.py [--n 30]

Order of launches after warm-up (kernel-name filter picks what to capture):
  1. k_sweep_high   : H on target n-10 (two-stream path)
  2. k_sweep_low    : H on target 3    (shuffle path)
  3. k_phase        : cu1 on (n-1, 7)
  4. k_fused        : first pass of the fused H layer, interpreted (QSB_FUSED_JIT=0)
  5. qsb_pass       : the same pass compiled at run time (jit.cu)
  6. qsb_pass       : first pass of QFT(n), compiled
  7. k_sweep_high_d : H on target n-11 of an (n-1)-qubit complex128 register
  8. k_probs / chunk_sums / k_trajectories / k_resolve / k_draws : probabilities + 10^5 samples
"""
import argparse
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_1805_00988_b200 import State, build_hadamard_layer, build_qft, fusion, u1  # noqa: E402
from paper_1805_00988_b200.circuits import lower_ops  # noqa: E402
from paper_1805_00988_b200.gates import H  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=30)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
n = a.n
st = State(n)
passes = fusion.plan(n, lower_ops(build_hadamard_layer(n)))
qpasses = fusion.plan(n, lower_ops(build_qft(n)))
for _ in range(a.reps):
    st.apply_gate(H, n - 10)
    st.apply_gate(H, 3)
    st.apply_controlled_gate(u1(0.5), n - 1, 7)
    os.environ["QSB_FUSED_JIT"] = "0"
    st.apply_fused(passes[0].tile, passes[0].op_array())
    os.environ["QSB_FUSED_JIT"] = "2"
    st.apply_fused(passes[0].tile, passes[0].op_array())
    st.apply_fused(qpasses[0].tile, qpasses[0].op_array())
st.flush()
sd = State(n - 1, precision="double")
sd.apply_gate(H, n - 11)
sd.flush()
sd.close()
st.probabilities(0, 1 << 24)
st.sample_outcomes(100_000, 3)
print("profiled kernels launched", len(passes), "H-layer passes,", len(qpasses), "QFT passes")
