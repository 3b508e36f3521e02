"""Sharded registers across PROCESSES on the GPU box: 2 and 4 ranks on the one
B200, gloo for the control plane, the data plane through cudaIpc-mapped peer
memory (qs_ipc_open: the partner's shard mapped into this process; same-device
IPC works across processes).  Qubit swaps run qs_swap_peer, global-target
gates (peer_gates=True) qs_apply_gate_peer — the kernels the multi-GPU path
runs over NVLink.  Results must equal the unsharded register bit for bit
(values), probabilities byte for byte and sampled outcomes draw for draw.

(NCCL cannot put two ranks on one GPU, so the NCCL send/recv exchange is
covered by the gloo CPU tests in test_sharded.py and by bench.py --gpus N on
multi-GPU boxes.)
"""

from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _circuit(n, seed):
    from paper_1805_00988_b200 import Circuit, build_hadamard_layer, build_qft
    from test_sharded import mixed_circuit

    return Circuit(n, build_hadamard_layer(n).instructions + mixed_circuit(n, 120, seed).instructions
                   + build_qft(n).instructions[-60:])


def _worker(rank, world, port, n, seed, peer_gates, q):
    import sys
    from pathlib import Path

    here = Path(__file__).resolve().parent
    sys.path[:0] = [str(here), str(here.parent)]
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_00988_b200.sharded import ShardedState

        circ = _circuit(n, seed)
        st = ShardedState.distributed(n, device=0, peer_gates=peer_gates, exchange="peer")
        st.run(circ)
        # more gates through the per-gate API, global targets included
        for t in range(n - 3, n):
            st.h(t)
            st.cx(0, t)
        amps = st.amplitudes()
        probs = st.probabilities()
        draws = st.sample_outcomes(4000, seed)
        info = (st.exchange, st.swaps, st.peer_swaps, st.peer_gate_count)
        st.close()
        if rank == 0:
            from paper_1805_00988_b200 import State, execute

            ref = State(n)
            execute(circ, ref, fuse=False)
            for t in range(n - 3, n):
                ref.h(t)
                ref.cx(0, t)
            ra = ref.amplitudes()
            q.put((bool(np.all(amps == ra)), probs.tobytes() == ref.probabilities().tobytes(),
                   bool(np.array_equal(draws, ref.sample_outcomes(4000, seed))), info))
            ref.close()
    except Exception as exc:  # noqa: BLE001
        q.put(("error", rank, repr(exc)))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,peer_gates", [(2, 18, False), (2, 18, True), (4, 19, False), (4, 19, True)])
def test_processes_share_shards_over_peer_memory(world, n, peer_gates):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, 100 + n, peer_gates, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    codes = [p.exitcode for p in procs]
    res = q.get(timeout=10)
    assert res[0] != "error", res
    assert all(c == 0 for c in codes), codes
    amps_ok, probs_ok, draws_ok, (mode, swaps, peer_swaps, peer_gate_count) = res
    assert mode == "peer" and peer_swaps == swaps
    assert peer_gate_count > 0 if peer_gates else swaps > 0
    assert amps_ok and probs_ok and draws_ok
