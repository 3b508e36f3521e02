"""Sharded-register host logic on the CPU (gloo, world size 2 and 4; virtual
shards), with the oracle as the per-shard engine.  The same ShardedState code
drives libqsb200 shards over NCCL on GPUs (tests/test_gpu_sharded.py)."""

from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from golden_util import M8Gate, same_values
from oracle import c as oc
from paper_1805_00988_b200 import FIXED_GATES, Circuit, build_hadamard_layer, build_qft, random_circuit, u1
from paper_1805_00988_b200.circuits import Apply, ControlledApply, ControlledControlledApply
from paper_1805_00988_b200.sharded import QubitLayout, ShardedState, exchange_plan
from shard_engines import OracleEngine


def oracle_run(circuit, basis=0):
    amps = np.zeros(1 << circuit.num_qubits, np.complex64)
    amps[basis] = 1
    for ins in circuit.instructions:
        if isinstance(ins, Apply):
            oc.apply_gate(amps, ins.target, ins.gate)
        elif isinstance(ins, ControlledApply):
            oc.apply_controlled_gate(amps, ins.control, ins.target, ins.gate)
        elif isinstance(ins, ControlledControlledApply):
            oc.apply_cc_gate(amps, ins.control1, ins.control2, ins.target, ins.gate)
    return amps


def mixed_circuit(n, depth, seed):
    rng = np.random.default_rng(seed)
    circ = random_circuit(n, depth, rng)
    extra = []
    for _ in range(depth // 8):
        c1, c2, t = (int(x) for x in rng.choice(n, 3, replace=False))
        extra.append(ControlledControlledApply(FIXED_GATES["x"], c1, c2, t))
    ins = list(circ.instructions)
    for k, e in enumerate(extra):
        ins.insert((k * 7) % (len(ins) + 1), e)
    return Circuit(n, tuple(ins))


class TestLayout:
    def test_swap_bookkeeping(self):
        lay = QubitLayout(6, 2)
        lay.swap_physical(5, 3)
        assert lay.pos[5] == 3 and lay.pos[3] == 5 and lay.at[3] == 5 and lay.at[5] == 3
        assert not lay.is_local(3) and lay.is_local(5)
        phys = np.arange(64)
        log = lay.logical_of_physical_index(phys)
        assert sorted(log.tolist()) == list(range(64))
        assert log[1 << 3] == 1 << 5

    def test_exchange_plan_halves(self):
        L = 5
        for rb in range(3):
            for r in range(8):
                partner, off, cnt = exchange_plan(r, rb, L)
                assert partner == r ^ (1 << rb) and cnt == 16
                assert off == (16 if not (r >> rb) & 1 else 0)
                # partners exchange complementary halves
                assert exchange_plan(partner, rb, L)[1] == 16 - off

    def test_exchange_is_the_bit_swap(self):
        """Swapping halves by exchange_plan == permuting index bits L-1 <-> L+b."""
        n, g = 6, 2
        L = n - g
        full = np.arange(1 << n).astype(np.complex64)
        shards = [full[r << L:(r + 1) << L].copy() for r in range(1 << g)]
        b = 1
        for r in range(1 << g):
            p, off, cnt = exchange_plan(r, b, L)
            if p < r:
                continue
            _, poff, _ = exchange_plan(p, b, L)
            tmp = shards[r][off:off + cnt].copy()
            shards[r][off:off + cnt] = shards[p][poff:poff + cnt]
            shards[p][poff:poff + cnt] = tmp
        got = np.concatenate(shards)
        idx = np.arange(1 << n)
        s, t = L - 1, L + b
        bs, bt = (idx >> s) & 1, (idx >> t) & 1
        src = idx ^ ((bs ^ bt) << s) ^ ((bs ^ bt) << t)
        assert np.array_equal(got, full[src])


class TestVirtualShards:
    @pytest.mark.parametrize("n,shards", [(6, 2), (7, 4), (8, 8), (9, 4)])
    def test_random_circuits_bitwise(self, n, shards):
        for seed in range(3):
            circ = mixed_circuit(n, 60, seed + 10 * n)
            ref = oracle_run(circ)
            st = ShardedState.virtual(n, shards, engine_factory=OracleEngine)
            st.run(circ)
            assert same_values(st.amplitudes(), ref)
            assert abs(st.norm_squared() - float(oc.probabilities(ref).sum())) < 1e-12
            assert st.probabilities().tobytes() == oc.probabilities(ref).tobytes()

    def test_gate_api_matches_run(self):
        n, shards = 7, 4
        circ = mixed_circuit(n, 40, 99)
        a = ShardedState.virtual(n, shards, engine_factory=OracleEngine)
        for ins in circ.instructions:
            if isinstance(ins, Apply):
                a.apply_gate(ins.gate, ins.target)
            elif isinstance(ins, ControlledApply):
                a.apply_controlled_gate(ins.gate, ins.control, ins.target)
            else:
                a.apply_controlled_controlled_gate(ins.gate, ins.control1, ins.control2, ins.target)
        assert same_values(a.amplitudes(), oracle_run(circ))

    def test_hlayer_and_qft_global_qubits(self):
        n, shards = 8, 4
        circ = Circuit(n, build_hadamard_layer(n).instructions + build_qft(n).instructions)
        st = ShardedState.virtual(n, shards, engine_factory=OracleEngine)
        st.run(circ)
        assert st.swaps >= 2  # both global qubits were swapped in
        assert same_values(st.amplitudes(), oracle_run(circ))

    @pytest.mark.parametrize("n,shards", [(6, 2), (8, 4), (9, 8)])
    def test_sampling_matches_unsharded(self, n, shards):
        """The exact CDF is chained across shard boundaries: same draws as pairsim."""
        circ = mixed_circuit(n, 50, 7 * n)
        ref = oracle_run(circ)
        st = ShardedState.virtual(n, shards, engine_factory=OracleEngine)
        st.run(circ)
        for seed in (0, 5, 123):
            got = st.sample_outcomes(4000, seed)
            assert np.array_equal(got, oc.sample_outcomes(ref, 4000, seed))
        m = st.measure_collapse(seed=9)
        assert m == int(oc.sample_outcomes(ref, 1, 9)[0])
        a = st.amplitudes()
        assert a[m] == 1 and np.count_nonzero(a) == 1

    def test_sampling_zero_probability_shards(self):
        n = 7
        st = ShardedState.virtual(n, 4, engine_factory=OracleEngine)
        st.reset(0b1011011)  # all probability in shard 2
        assert np.all(st.sample_outcomes(100, 3) == 0b1011011)

    def test_reset_basis_on_other_shard(self):
        n = 6
        st = ShardedState.virtual(n, 4, engine_factory=OracleEngine)
        st.reset(0b110101)
        a = st.amplitudes()
        assert a[0b110101] == 1 and np.count_nonzero(a) == 1


class TestPeerGates:
    """Global-target gates as one peer-memory update per partner pair
    (csrc/peer.cu semantics, oracle engines): no qubit swaps, same bits."""

    @pytest.mark.parametrize("n,shards", [(6, 2), (7, 4), (8, 8), (9, 4)])
    def test_random_circuits_bitwise(self, n, shards):
        for seed in range(3):
            circ = mixed_circuit(n, 60, seed + 10 * n)
            ref = oracle_run(circ)
            st = ShardedState.virtual(n, shards, engine_factory=OracleEngine, peer_gates=True)
            st.run(circ)
            assert st.peer_gate_count > 0
            assert same_values(st.amplitudes(), ref)

    def test_gate_api_and_controls_on_every_bit_class(self):
        """Controls on local bits (including the split bit's neighbours), on other
        global bits (rank predicates), and all-local-controlled targets."""
        n, shards = 6, 4
        rng = np.random.default_rng(3)
        ins = [Apply(FIXED_GATES["h"], q) for q in range(n)]
        for _ in range(40):
            t = int(rng.integers(n - 2, n))  # global targets
            others = [q for q in range(n) if q != t]
            g = [FIXED_GATES["h"], FIXED_GATES["x"], FIXED_GATES["y"], u1(0.7)][int(rng.integers(4))]
            k = rng.random()
            if k < 0.3:
                ins.append(Apply(g, t))
            elif k < 0.7:
                ins.append(ControlledApply(g, int(rng.choice(others)), t))
            else:
                c1, c2 = (int(x) for x in rng.choice(others, 2, replace=False))
                ins.append(ControlledControlledApply(g, c1, c2, t))
        circ = Circuit(n, tuple(ins))
        st = ShardedState.virtual(n, shards, engine_factory=OracleEngine, peer_gates=True)
        for i in circ.instructions:
            if isinstance(i, Apply):
                st.apply_gate(i.gate, i.target)
            elif isinstance(i, ControlledApply):
                st.apply_controlled_gate(i.gate, i.control, i.target)
            else:
                st.apply_controlled_controlled_gate(i.gate, i.control1, i.control2, i.target)
        assert st.peer_gate_count > 0
        assert same_values(st.amplitudes(), oracle_run(circ))

    def test_hlayer_and_qft_without_swaps(self):
        n, shards = 8, 4
        circ = Circuit(n, build_hadamard_layer(n).instructions + build_qft(n).instructions)
        st = ShardedState.virtual(n, shards, engine_factory=OracleEngine, peer_gates=True)
        st.run(circ)
        # only the all-global controlled phase cu1(7, 6) still swaps a qubit in
        assert st.swaps <= 1 and st.peer_gate_count >= 2
        assert same_values(st.amplitudes(), oracle_run(circ))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class TestPeerExchange:
    """Qubit swaps moved by qs_swap_peer semantics (partners split the
    exchanged half between them; oracle engines) == the oracle, bitwise."""

    @pytest.mark.parametrize("n,shards", [(6, 2), (7, 4), (8, 8)])
    def test_random_circuits_bitwise(self, n, shards):
        for seed in range(3):
            circ = mixed_circuit(n, 60, seed + 7 * n)
            ref = oracle_run(circ)
            st = ShardedState.virtual(n, shards, engine_factory=OracleEngine, exchange="peer")
            st.run(circ)
            assert st.peer_swaps > 0 and st.peer_swaps == st.swaps
            assert same_values(st.amplitudes(), ref)

    def test_peer_gates_and_peer_swaps_together(self):
        n, shards = 7, 4
        circ = mixed_circuit(n, 80, 99)
        st = ShardedState.virtual(n, shards, engine_factory=OracleEngine, peer_gates=True, exchange="peer")
        st.run(circ)
        st.canonicalize()  # readout swaps go through the peer exchange too
        assert same_values(st.amplitudes(), oracle_run(circ))

    def test_bad_mode(self):
        with pytest.raises(ValueError):
            ShardedState.virtual(5, 2, engine_factory=OracleEngine, exchange="carrier-pigeon")


def _worker(rank, world, port, n, seed, q, peer=False, chunk=1 << 26):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        circ = mixed_circuit(n, 50, seed)
        # peer=True: oracle engines cannot map a partner process's buffer, so
        # every rank must agree to fall back to qubit swaps (no rank waits)
        st = ShardedState.distributed(n, engine_factory=OracleEngine, peer_gates=peer)
        st.chunk = chunk  # small chunks: the double-buffered send/recv loop
        st.run(circ)
        amps = st.amplitudes()
        probs = st.probabilities()
        norm = st.norm_squared()
        draws = st.sample_outcomes(3000, seed)
        if rank == 0:
            ref = oracle_run(circ)
            q.put((bool(same_values(amps, ref)), probs.tobytes() == oc.probabilities(ref).tobytes(),
                   abs(norm - float(oc.probabilities(ref).sum())) < 1e-12, st.swaps,
                   bool(np.array_equal(draws, oc.sample_outcomes(ref, 3000, seed)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,peer,chunk", [(2, 7, False, 1 << 26), (4, 8, False, 1 << 26), (2, 7, True, 1 << 26),
                                               (2, 8, False, 8), (4, 8, False, 4)])
def test_gloo_distributed_matches_oracle(world, n, peer, chunk):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, 1234 + n, q, peer, chunk)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    assert all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    amps_ok, probs_ok, norm_ok, swaps, draws_ok = q.get(timeout=5)
    assert amps_ok and probs_ok and norm_ok and swaps > 0 and draws_ok


def test_all_global_diagonal_gates_need_no_exchange():
    """A diagonal gate whose bits are all global multiplies whole shards in
    place (no qubit swap), with the oracle's values."""
    n, shards = 7, 4
    basis = (1 << (n - 1)) | (1 << (n - 2)) | 5
    ins = (ControlledApply(u1(0.37), n - 1, n - 2), Apply(FIXED_GATES["t"], n - 1),
           ControlledApply(FIXED_GATES["s"], n - 2, n - 1), Apply(FIXED_GATES["h"], 0))
    circ = Circuit(n, ins)
    for use_run in (False, True):
        st = ShardedState.virtual(n, shards, engine_factory=OracleEngine)
        st.reset(basis)
        if use_run:
            st.run(circ)
        else:
            for i in ins:
                if isinstance(i, Apply):
                    st.apply_gate(i.gate, i.target)
                else:
                    st.apply_controlled_gate(i.gate, i.control, i.target)
        assert st.shard_phases == 3 and st.swaps == 0
        assert same_values(st.amplitudes(), oracle_run(circ, basis))


def test_auto_global_gate_mode_calibrates_and_keeps_bits():
    """peer_gates="auto": the first global-target pair gate times a peer gate
    against swap + sweep (X twice each: the register's bits and the qubit map
    are unchanged) and keeps the faster; results stay bit-exact."""
    n, shards = 8, 4
    circ = mixed_circuit(n, 80, 77)
    st = ShardedState.virtual(n, shards, engine_factory=OracleEngine, peer_gates="auto")
    st.run(circ)
    assert st.calibration is not None and st.calibration["chosen"] in ("peer", "swap")
    assert st.calibration["peer_gate_ms"] > 0 and st.calibration["swap_and_sweep_ms"] > 0
    assert same_values(st.amplitudes(), oracle_run(circ))
