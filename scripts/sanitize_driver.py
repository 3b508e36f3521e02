"""Small workloads for compute-sanitizer (memcheck / racecheck / synccheck):
the fused TMA tile kernel (interpreter k_fused and a compiled qsb_pass), the
sweep / phase kernels, the exact sampling chain (M1-M6) and the peer-memory
pair and swap kernels (virtual shards on one GPU).  n <= 16.

    compute-sanitizer --tool racecheck python scripts/sanitize_driver.py [part]
"""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import numpy as np  # noqa: E402

from paper_1805_00988_b200 import State, build_qft, fusion, layered_random_circuit, random_unitary_gate  # noqa: E402
from paper_1805_00988_b200.circuits import lower_ops  # noqa: E402

part = sys.argv[1] if len(sys.argv) > 1 else "all"
n = 14
rng = np.random.default_rng(7)

if part in ("all", "fused"):
    for jit in ("0", "2"):  # interpreter kernel, then a compiled program
        os.environ["QSB_FUSED_JIT"] = jit
        st = State(n)
        for q in range(n):
            st.h(q)
        for circ in (build_qft(n), layered_random_circuit(n, 3, seed=1)):
            fusion.run(st, fusion.plan(n, lower_ops(circ), 10))
        st.flush()
        st.close()
    os.environ["QSB_FUSED_JIT"] = "2"
    st = State(n)
    fusion.run(st, fusion.plan(n, lower_ops(build_qft(n)), 10), combine=True)
    st.flush()
    st.close()

if part in ("all", "sweeps"):
    st = State(n)
    g = random_unitary_gate(rng)
    for t in range(n):
        st.apply_gate(g, t)
    st.apply_controlled_gate(g, 3, 9)
    st.apply_controlled_controlled_gate(g, 0, 13, 6)
    st.cu1(11, 2, 0.3)
    st.swap_qubits(1, 12)
    st.flush()
    st.close()

if part in ("all", "sample"):
    st = State(n)
    for q in range(n):
        st.h(q)
    st.t(2)
    st.sample_outcomes(5000, 3)
    st.probabilities()
    st.norm_squared()
    st.measure_collapse(4)
    st.close()

if part in ("all", "sample18"):
    # n = 18: whole warps of 4096-amplitude chunks, so M3 takes the bulk-copy
    # ring (k_trajectories_bulk) and M4b the bulk-copied chunk re-sums
    m = 18
    st = State(m)
    for q in range(m):
        st.h(q)
    st.t(2)
    st.sample_outcomes(3000, 5)
    mag = np.exp(rng.uniform(np.log(1e-30), 0.0, size=1 << m))
    st.set_amplitudes((mag * np.exp(2j * np.pi * rng.random(1 << m))).astype(np.complex64))
    st.sample_outcomes(3000, 6)
    # a measured circuit: the reset folded into the first fused pass, the
    # sampler's row sums left by the last one (producer-warp epilogue)
    from paper_1805_00988_b200 import execute
    from paper_1805_00988_b200.circuits import Circuit, SampleMeasure

    execute(Circuit(m, build_qft(m).instructions + (SampleMeasure(2000),)), st, seed=7, initial_basis=5)
    st.close()

if part in ("all", "peer"):
    from paper_1805_00988_b200.sharded import ShardedState

    for peer, exch in ((True, "peer"), (False, "peer")):
        vs = ShardedState.virtual(n, 2, peer_gates=peer, exchange=exch)
        for q in range(n):
            vs.h(q)
        vs.cx(n - 1, 0)
        vs.amplitudes()
        vs.close()
if part in ("all", "multidev"):
    from paper_1805_00988_b200 import build_qft
    from paper_1805_00988_b200.multigpu import MultiDeviceState
    from paper_1805_00988_b200.sharded import ShardedState

    for peer in (False, True):
        with MultiDeviceState(n, [0, 0, 0, 0], peer_gates=peer) as md:
            for q in range(n):
                md.h(q)
            md.cx(n - 1, 0)
            md.run(build_qft(n), fuse=True)
            md.sample_outcomes(1000, 1)
            md.probabilities()
    vs = ShardedState.virtual(n, 2, peer_gates=True, exchange="peer", precision="double")
    for q in range(n):
        vs.h(q)
    vs.amplitudes()
    vs.close()
print("sanitize driver done:", part)
