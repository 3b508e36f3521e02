"""Registers sharded over P = 2^g GPUs on their top g qubits.

Layout: physical qubit positions 0..L-1 (L = n - g) are local index bits of
every shard; positions L..n-1 are the shard (rank) bits, so shard r owns the
contiguous slice [r * 2^L, (r+1) * 2^L) of the physical index space.  A
logical -> physical qubit map (QubitLayout) is kept on the host and updated
lazily:

* a gate whose target and controls are local runs on every shard with no
  communication; a control on a global qubit is a shard predicate (shards
  whose bit is 0 skip the gate);
* a gate targeting a global qubit first swaps that physical position with
  local position L-1 ("qubit swap"): partner shards r and r ^ (1 << b)
  exchange the half of their slice whose bit L-1 differs from their own
  rank bit b.  With s = L-1 that half is contiguous, so the exchange is two
  plain buffers (NCCL send/recv over NVLink, or an in-process copy for
  virtual shards) and needs no pack/unpack kernel.  No swap-back: the map
  records the permutation and readout un-permutes it (canonicalize()).

Transports:
* DistTransport  — one process per GPU, torch.distributed (NCCL on GPUs,
  gloo for the CPU tests), chunked through a staging buffer;
* LocalTransport — P virtual shards in one process (one GPU or CPU engines),
  the same swap logic with in-process copies.

The per-shard compute engine is pluggable: CudaEngine wraps a device State
(libqsb200); tests plug in an oracle engine on the CPU.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .gates import FIXED_GATES, m8, u1 as _u1


# ----------------------------------------------------------------------------
class QubitLayout:
    """Logical -> physical qubit positions for n qubits over 2^g shards."""

    def __init__(self, n: int, g: int):
        if g < 0 or g >= n:
            raise ValueError("need 0 <= g < n")
        self.n, self.g, self.L = n, g, n - g
        self.pos = list(range(n))  # pos[logical] = physical
        self.at = list(range(n))   # at[physical] = logical

    def is_local(self, q: int) -> bool:
        return self.pos[q] < self.L

    def swap_physical(self, p1: int, p2: int) -> None:
        a, b = self.at[p1], self.at[p2]
        self.at[p1], self.at[p2] = b, a
        self.pos[a], self.pos[b] = p2, p1

    def is_identity(self) -> bool:
        return self.pos == list(range(self.n))

    def logical_of_physical_index(self, phys: np.ndarray) -> np.ndarray:
        """Map physical basis indices to logical ones (bit at[p] <- bit p)."""
        phys = np.asarray(phys, dtype=np.int64)
        out = np.zeros_like(phys)
        for p in range(self.n):
            out |= ((phys >> p) & 1) << self.at[p]
        return out


def exchange_plan(rank: int, rank_bit: int, L: int) -> tuple[int, int, int]:
    """(partner, offset, count) for swapping physical position L + rank_bit
    with local position L-1: send/receive the contiguous half of the local
    slice whose bit L-1 differs from this rank's bit `rank_bit`."""
    partner = rank ^ (1 << rank_bit)
    rb = (rank >> rank_bit) & 1
    half = 1 << (L - 1)
    offset = half if rb == 0 else 0
    return partner, offset, half


# ----------------------------------------------------------------------------
class CudaEngine:
    """One shard on a GPU: a libqsb200 State of L qubits."""

    def __init__(self, num_qubits: int, device: int = 0, memory_budget: int | None = None,
                 precision: str = "single"):
        from .state import State

        self.state = State(num_qubits, device=device, memory_budget=memory_budget, precision=precision)
        self.num_qubits = num_qubits
        self.device = device
        self.double = self.state.is_double
        self.unit = 4 if self.double else 2  # float32 words per amplitude (exchange views)
        self._view = None

    def reset(self, basis: int | None) -> None:
        """e_basis, or the zero vector for basis=None (a shard not holding |basis>)."""
        self.state.reset(0 if basis is None else basis)
        if basis is None:
            self.state.set_amplitudes(np.zeros(1, np.complex128 if self.double else np.complex64), offset=0)

    def apply(self, kind: int, target: int, ctrl_mask: int, m: np.ndarray) -> None:
        from . import fusion

        fusion._single(self.state, kind, target, ctrl_mask, m)

    def apply_ops(self, ops, exact: bool = True) -> None:
        from . import fusion

        K = 12 if self.double else None  # complex128 tiles: 2^12 amplitudes (64 KiB)
        fusion.run(self.state, fusion.plan(self.num_qubits, ops, K, reorder=not exact), combine=not exact)

    def swap_qubits(self, a: int, b: int) -> None:
        self.state.swap_qubits(a, b)

    def view(self):
        """torch float32 view (unit * 2^L,) of the device amplitudes (zero-copy)."""
        import torch

        if self._view is None:
            ptr = self.state.device_pointer()
            nfloat = self.unit << self.num_qubits

            class _CAI:
                __cuda_array_interface__ = {"shape": (nfloat,), "typestr": "<f4", "data": (ptr, False),
                                            "version": 3, "strides": None}

            self._view = torch.as_tensor(_CAI(), device=torch.device("cuda", self.device))
        return self._view

    def comm_begin(self) -> None:
        """Order torch's stream after this shard's kernels."""
        import torch

        ext = torch.cuda.ExternalStream(self.state.stream(), device=torch.device("cuda", self.device))
        torch.cuda.current_stream(self.device).wait_stream(ext)

    def comm_end(self) -> None:
        """Order this shard's stream after torch's (copies / NCCL) work."""
        import torch

        ext = torch.cuda.ExternalStream(self.state.stream(), device=torch.device("cuda", self.device))
        ext.wait_stream(torch.cuda.current_stream(self.device))

    def amplitudes(self) -> np.ndarray:
        return self.state.amplitudes()

    def probabilities(self) -> np.ndarray:
        return self.state.probabilities()

    def close(self) -> None:
        self._view = None
        self.state.close()

    def norm_squared(self) -> float:
        return self.state.norm_squared()

    def synchronize(self) -> None:
        self.state.flush()

    def cdf_extend(self, start: float) -> float:
        return self.state.cdf_extend(start)

    def sample_shard(self, k, rng, start, total, base, gdim, is_last) -> np.ndarray:
        return self.state.sample_shard(k, rng, start, total, base, gdim, is_last)

    # ---- peer-memory global gates (csrc/peer.cu) --------------------------------
    def peer_ref(self):
        """What a partner in this process passes to peer_gate: our device pointer."""
        return self.state.device_pointer()

    def ipc_handle(self) -> bytes:
        import ctypes

        buf = ctypes.create_string_buffer(64)
        N.check(N.lib().qs_ipc_handle(self.state.handle, buf))
        return buf.raw

    def open_peer(self, handle: bytes) -> int:
        import ctypes

        ptr = ctypes.c_void_p()
        N.check(N.lib().qs_ipc_open(self.device, handle, ctypes.byref(ptr)))
        return ptr.value

    def close_peer(self, ptr: int) -> None:
        N.lib().qs_ipc_close(self.device, ptr)

    def swap_peer(self, peer, own_off: int, peer_off: int, count: int) -> None:
        N.check(N.lib().qs_swap_peer(self.state.handle, peer, int(own_off), int(peer_off), int(count)))

    def peer_gate(self, peer, own_is_a: bool, ctrl_mask: int, m: np.ndarray) -> None:
        if m.dtype == np.float64:
            mm = np.ascontiguousarray(m)
            N.check(N.lib().qs_apply_gate_peer_f64(self.state.handle, peer, int(bool(own_is_a)), int(ctrl_mask),
                                                   N.f64ptr(mm)))
            return
        mm = np.ascontiguousarray(m, dtype=np.float32)
        N.check(N.lib().qs_apply_gate_peer(self.state.handle, peer, int(bool(own_is_a)), int(ctrl_mask),
                                           N.f32ptr(mm)))


# ----------------------------------------------------------------------------
class LocalTransport:
    """All shards live in this process (virtual shards)."""

    def __init__(self, world: int):
        self.world = world

    def exchange(self, engines, rank_bit: int, L: int, chunk: int) -> None:
        for r in range(len(engines)):
            partner, off, cnt = exchange_plan(r, rank_bit, L)
            if partner < r:
                continue
            _, poff, _ = exchange_plan(partner, rank_bit, L)
            a, b = engines[r], engines[partner]
            a.comm_begin()
            b.comm_begin()
            va, vb = a.view(), b.view()
            u = getattr(a, "unit", 2)  # float32 words per amplitude
            sa = va[u * off: u * (off + cnt)]
            sb = vb[u * poff: u * (poff + cnt)]
            tmp = sa.clone()
            sa.copy_(sb)
            sb.copy_(tmp)
            a.comm_end()
            b.comm_end()

    def allreduce_sum(self, values):
        return [sum(values)] * len(values)

    def peer_setup(self, engines, ranks, g):
        """{(rank, partner): partner's peer reference} for every rank bit."""
        by_rank = dict(zip(ranks, engines))
        return {(r, r ^ (1 << b)): by_rank[r ^ (1 << b)].peer_ref() for r in ranks for b in range(g)}

    def peer_barrier(self, engines):
        for eng in engines:
            eng.synchronize()

    def cdf_chain(self, engines, ranks):
        """Exact running-sum entry value of every shard, in rank order."""
        starts, s = {}, 0.0
        for eng, r in sorted(zip(engines, ranks), key=lambda x: x[1]):
            starts[r] = s
            s = eng.cdf_extend(s)
        return starts, s

    def combine_max(self, arrays):
        return np.maximum.reduce(arrays)

    def common_seed_words(self, seed):
        return N.pcg_from_seed(seed)


class DistTransport:
    """One shard per process; torch.distributed point-to-point exchange."""

    def __init__(self, group=None):
        import torch.distributed as dist

        self.dist = dist
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self._staging = None
        # send/recv of device tensors needs NCCL; a gloo control plane with
        # CUDA shards moves data through mapped peer memory instead
        self.moves_device_buffers = dist.get_backend(group) == "nccl"

    def exchange(self, engines, rank_bit: int, L: int, chunk: int) -> None:
        """NCCL send/recv of the half-shard in chunks through two staging
        buffers: chunk k+1's transfer is in flight while chunk k is copied
        into place (the send of a chunk and the receive into the same
        addresses cannot alias, hence the staging)."""
        dist = self.dist
        (eng,) = engines
        partner, off, cnt = exchange_plan(self.rank, rank_bit, L)
        eng.comm_begin()
        v = eng.view()
        u = getattr(eng, "unit", 2)  # float32 words per amplitude
        step = min(cnt, chunk)
        nbuf = 2 if cnt > step else 1
        if self._staging is None or self._staging.numel() < u * step * nbuf or self._staging.device != v.device:
            self._staging = v.new_empty(u * step * nbuf)
        peer = dist.get_global_rank(self.group, partner) if self.group is not None else partner
        starts = list(range(off, off + cnt, step))

        def post(i):
            c = starts[i]
            mine = v[u * c: u * (c + step)]
            stg = self._staging[u * step * (i % nbuf): u * step * (i % nbuf + 1)]
            ops = [dist.P2POp(dist.isend, mine, peer, self.group), dist.P2POp(dist.irecv, stg, peer, self.group)]
            return dist.batch_isend_irecv(ops), mine, stg

        cur = post(0)
        for i in range(len(starts)):
            # posted after chunk i-1's copy-back (stream order protects its
            # staging buffer), before chunk i's
            nxt = post(i + 1) if i + 1 < len(starts) else None
            works, mine, stg = cur
            for w in works:
                w.wait()
            mine.copy_(stg)
            cur = nxt
        eng.comm_end()

    def peer_setup(self, engines, ranks, g):
        """Map the partner shards' buffers into this process (cudaIpc over
        NVLink).  All ranks agree on success (a MIN all-reduce), so a rank that
        cannot map its partners never leaves the others waiting: on failure
        every rank returns None and the swap path is used."""
        import torch

        (eng,) = engines
        handles = [None] * self.world
        ok = 1
        try:
            mine = eng.ipc_handle()
        except Exception:  # noqa: BLE001
            mine, ok = b"", 0
        self.dist.all_gather_object(handles, mine, group=self.group)
        peers = {}
        if ok:
            try:
                for b in range(g):
                    partner = self.rank ^ (1 << b)
                    peers[(self.rank, partner)] = eng.open_peer(handles[partner])
            except Exception:  # noqa: BLE001
                ok = 0
        flag = self._tensor(torch.tensor([ok], dtype=torch.int32))
        self.dist.all_reduce(flag, op=self.dist.ReduceOp.MIN, group=self.group)
        if int(flag.cpu().item()) != 1:
            for ptr in peers.values():
                eng.close_peer(ptr)
            return None
        return peers

    def peer_barrier(self, engines):
        (eng,) = engines
        eng.synchronize()
        self.dist.barrier(group=self.group)

    def _tensor(self, arr):
        import torch

        t = torch.as_tensor(arr)
        return t.cuda() if self.dist.get_backend(self.group) == "nccl" else t

    def _peer(self, r):
        return self.dist.get_global_rank(self.group, r) if self.group is not None else r

    def cdf_chain(self, engines, ranks):
        """Rank r waits for rank r-1's exact end value, extends it over its own
        shard and passes it on; the last rank's end is broadcast as the total."""
        import torch

        (eng,) = engines
        start = torch.zeros(1, dtype=torch.float64)
        if self.rank > 0:
            t = self._tensor(start)
            self.dist.recv(t, self._peer(self.rank - 1), group=self.group)
            start = t.cpu()
        s0 = float(start.item())
        end = eng.cdf_extend(s0)
        if self.rank < self.world - 1:
            self.dist.send(self._tensor(torch.tensor([end], dtype=torch.float64)), self._peer(self.rank + 1),
                           group=self.group)
        tot = self._tensor(torch.tensor([end], dtype=torch.float64))
        self.dist.broadcast(tot, self._peer(self.world - 1), group=self.group)
        return {self.rank: s0}, float(tot.cpu().item())

    def combine_max(self, arrays):
        import torch

        (a,) = arrays
        t = self._tensor(torch.from_numpy(a.copy()))
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX, group=self.group)
        return t.cpu().numpy()

    def common_seed_words(self, seed):
        """Every rank must draw from the same generator: rank 0's state wins."""
        obj = [N.pcg_from_seed(seed)] if self.rank == 0 else [None]
        words = [(obj[0].state_hi, obj[0].state_lo, obj[0].inc_hi, obj[0].inc_lo)] if self.rank == 0 else [None]
        self.dist.broadcast_object_list(words, src=self._peer(0), group=self.group)
        return N.qs_pcg64(*words[0])

    def allreduce_sum(self, values):
        import torch

        (x,) = values
        t = torch.tensor([x], dtype=torch.float64)
        if self.dist.get_backend(self.group) == "nccl":
            t = t.cuda()
        self.dist.all_reduce(t, group=self.group)
        return [float(t.item())]


# ----------------------------------------------------------------------------
class ShardedState:
    """A 2^n register over 2^g shards (QCGPU-style gate API)."""

    def __init__(self, num_qubits: int, engines, transport, ranks, world: int,
                 chunk_amps: int = 1 << 26, peer_gates: bool | None = None, exchange: str | None = None):
        g = int(round(math.log2(world)))
        if 1 << g != world:
            raise ValueError("the shard count must be a power of two")
        if chunk_amps < 1 or chunk_amps & (chunk_amps - 1):
            # exchange chunks must tile the 2^(L-1)-amplitude half exactly, or
            # the partners' send / receive sizes would differ
            raise ValueError("chunk_amps must be a power of two")
        self.num_qubits = num_qubits
        self.layout = QubitLayout(num_qubits, g)
        self.engines = list(engines)
        self.ranks = list(ranks)  # rank id of each local engine
        self.transport = transport
        self.world = world
        self.chunk = chunk_amps
        self.swaps = 0
        # Global-target pair gates as one peer-memory kernel per partner pair
        # (csrc/peer.cu) instead of a qubit swap; QSB_SHARD_PEER=1 turns it on
        # by default.  Falls back to swaps if the partners cannot be mapped.
        if peer_gates is None:
            import os

            env = os.environ.get("QSB_SHARD_PEER", "0")
            peer_gates = "auto" if env == "auto" else env == "1"
        can_peer = g > 0 and all(hasattr(e, "peer_gate") for e in self.engines)
        # "auto": decided at the first global-target pair gate by timing both
        # paths on the live register (calibrate_global_gates)
        self._auto_peer = peer_gates == "auto" and can_peer
        self.peer_gates = (self._auto_peer or (peer_gates != "auto" and bool(peer_gates))) and can_peer
        self.calibration = None
        # Qubit-swap data movement: "nccl" (transport send/recv; in-process
        # copies for virtual shards) or "peer" (qs_swap_peer: one kernel per
        # partner over mapped peer memory, no staging).  Default: "peer" when
        # the transport cannot move device buffers itself (gloo control
        # plane with CUDA shards), else QSB_SHARD_EXCHANGE or "nccl".
        if exchange is None:
            import os

            exchange = os.environ.get("QSB_SHARD_EXCHANGE") or ("peer" if can_peer and not getattr(
                transport, "moves_device_buffers", True) else "nccl")
        if exchange not in ("nccl", "peer"):
            raise ValueError("exchange must be 'nccl' or 'peer'")
        self.exchange = exchange if can_peer else "nccl"
        self._peers = None
        self.peer_gate_count = 0
        self.peer_swaps = 0
        self.shard_phases = 0
        self.double = bool(getattr(self.engines[0], "double", False)) if self.engines else False

    def _m8(self, gate) -> np.ndarray:
        """Gate entries rounded to the shards' precision (kernel.py:118-119)."""
        from .gates import m8_for

        return m8_for(gate, self.double)

    # ---- constructors ------------------------------------------------------
    @classmethod
    def distributed(cls, num_qubits: int, group=None, device: int | None = None, engine_factory=None,
                    peer_gates: bool | None = None, memory_budget: int | None = None, exchange: str | None = None,
                    precision: str = "single"):
        import torch.distributed as dist

        tr = DistTransport(group)
        g = int(round(math.log2(tr.world)))
        L = num_qubits - g
        if engine_factory is None:
            import torch

            dev = torch.cuda.current_device() if device is None else device
            eng = CudaEngine(L, dev, memory_budget=memory_budget, precision=precision)
        else:
            eng = engine_factory(L)
        st = cls(num_qubits, [eng], tr, [tr.rank], tr.world, peer_gates=peer_gates, exchange=exchange)
        st.reset(0)
        return st

    @classmethod
    def virtual(cls, num_qubits: int, shards: int, device: int = 0, engine_factory=None,
                peer_gates: bool | None = None, memory_budget: int | None = None, exchange: str | None = None,
                precision: str = "single"):
        g = int(round(math.log2(shards)))
        L = num_qubits - g
        make = engine_factory or (lambda L_: CudaEngine(L_, device, memory_budget=memory_budget,
                                                        precision=precision))
        engines = [make(L) for _ in range(shards)]
        st = cls(num_qubits, engines, LocalTransport(shards), list(range(shards)), shards, peer_gates=peer_gates,
                 exchange=exchange)
        st.reset(0)
        return st

    # ---- state ----------------------------------------------------------------
    @property
    def L(self) -> int:
        return self.layout.L

    def reset(self, basis: int = 0) -> "ShardedState":
        """|basis> with the identity qubit map."""
        self.layout = QubitLayout(self.num_qubits, self.layout.g)
        owner, local = basis >> self.L, basis & ((1 << self.L) - 1)
        for eng, r in zip(self.engines, self.ranks):
            eng.reset(local if r == owner else None)
        return self

    # ---- gates ------------------------------------------------------------------
    def _exchange(self, rank_bit: int) -> None:
        """Swap physical positions L + rank_bit and L - 1 (data movement only;
        the caller updates the qubit map)."""
        if self.exchange == "peer" and self.L >= 2 and self._peer_ready():
            self._peer_swap(rank_bit)
        else:
            self.transport.exchange(self.engines, rank_bit, self.L, self.chunk)

    def _peer_swap(self, rank_bit: int) -> None:
        """The exchange of exchange_plan over peer memory: partners trade the
        halves whose bit L-1 differs from their rank bit, each moving half of
        that range with one qs_swap_peer kernel (no staging, no copy-back)."""
        L = self.L
        half = 1 << (L - 1)
        part = half // 2
        self.transport.peer_barrier(self.engines)
        for eng, r in zip(self.engines, self.ranks):
            partner, off, _ = exchange_plan(r, rank_bit, L)
            _, poff, _ = exchange_plan(partner, rank_bit, L)
            sub = part if (r >> rank_bit) & 1 else 0
            eng.swap_peer(self._peers[(r, partner)], off + sub, poff + sub, part)
        self.transport.peer_barrier(self.engines)
        self.peer_swaps += 1

    def _ensure_local(self, target: int) -> None:
        lay = self.layout
        if lay.is_local(target):
            return
        p = lay.pos[target]
        self._exchange(p - lay.L)
        lay.swap_physical(p, lay.L - 1)
        self.swaps += 1

    def _control_masks(self, controls) -> tuple[int, int]:
        """(local control mask, rank-bit predicate) under the current qubit map."""
        lay = self.layout
        cmask, need = 0, 0
        for c in controls:
            pc = lay.pos[c]
            if pc < lay.L:
                cmask |= 1 << pc
            else:
                need |= 1 << (pc - lay.L)
        return cmask, need

    def _peer_ready(self) -> bool:
        if not (self.peer_gates or self.exchange == "peer"):
            return False
        if self._peers is None:
            self._peers = self.transport.peer_setup(self.engines, self.ranks, self.layout.g) or False
            if self._peers is False:  # every rank agreed: fall back to transport swaps
                self.peer_gates = False
                self.exchange = "nccl"
        return bool(self._peers)

    def _global_pair_via_peer(self, rank_bit: int) -> bool:
        """Should a pair gate on global rank bit `rank_bit` run as a peer gate?"""
        if not (self.peer_gates and self._peer_ready()):
            return False
        if self._auto_peer and self.calibration is None:
            self.calibrate_global_gates(rank_bit)
        return self.peer_gates

    def calibrate_global_gates(self, rank_bit: int, reps: int = 1) -> dict:
        """Time both ways of a global-target pair gate on the live register and
        keep the faster (all ranks agree: max over ranks): a peer gate (one
        kernel over NVLink) vs a qubit swap + local sweep.  Uses X twice per
        path — an exact permutation, so the register's bits are unchanged
        and the qubit map is restored."""
        import time

        from .gates import FIXED_GATES

        X = self._m8(FIXED_GATES["x"])
        L = self.L

        def timed(fn):
            self.transport.peer_barrier(self.engines)
            t0 = time.perf_counter()
            for _ in range(reps):
                fn()
                fn()
            self.transport.peer_barrier(self.engines)
            return (time.perf_counter() - t0) / (2 * reps)

        def peer_once():
            self._peer_gate(rank_bit, 0, 0, X)
            self.peer_gate_count -= 1

        def swap_once():  # (exchange + sweep) twice: X X on the swapped-in qubit, then swap back
            self._exchange(rank_bit)
            for _ in range(2):
                for eng in self.engines:
                    eng.apply(N.QS_OP_PAIR, L - 1, 0, X)
            self._exchange(rank_bit)

        counters = (self.peer_swaps,)
        t_peer = timed(peer_once)
        # the swap's data movement both ways when the transport can move
        # device buffers itself (NCCL send/recv with staging) and the peers
        # are mapped (one swap kernel, no staging): the faster one becomes
        # the register's exchange
        modes = ["peer", "nccl"] if getattr(self.transport, "moves_device_buffers", True) else [self.exchange]
        keep = self.exchange
        t_modes = []
        for mode in modes:
            self.exchange = mode
            t_modes.append(timed(swap_once) / 2)  # one call = two (exchange + sweep)
        self.exchange = keep
        (self.peer_swaps,) = counters
        t = self.transport.combine_max([np.array([t_peer] + t_modes)])
        t_peer, t_modes = float(t[0]), [float(x) for x in t[1:]]
        best = int(np.argmin(t_modes))
        self.exchange = modes[best]
        t_swap = t_modes[best]
        self.peer_gates = t_peer <= t_swap
        self.calibration = {"peer_gate_ms": t_peer * 1e3, "swap_and_sweep_ms": t_swap * 1e3,
                            "swap_exchange": self.exchange,
                            **{f"swap_and_sweep_{m}_ms": x * 1e3 for m, x in zip(modes, t_modes)},
                            "chosen": "peer" if self.peer_gates else "swap"}
        return self.calibration

    def _shard_phase(self, rank_bits, m: np.ndarray) -> None:
        """A diagonal gate whose bits are all global: every amplitude of the
        shards whose rank bits are all 1 is multiplied by d — no exchange.
        Applied as the pair sweep of diag(d, d) (v_a' = d v_a + 0 v_b, the
        same product bit for bit up to the sign of zero)."""
        need = 0
        for b in rank_bits:
            need |= 1 << b
        dd = np.zeros(8, m.dtype)
        dd[0], dd[1], dd[6], dd[7] = m[6], m[7], m[6], m[7]
        for eng, r in zip(self.engines, self.ranks):
            if (r & need) == need:
                eng.apply(N.QS_OP_PAIR, 0, 0, dd)
        self.shard_phases += 1

    def _peer_gate(self, rank_bit: int, cmask: int, need: int, m: np.ndarray) -> None:
        """Pair update with the target on global rank bit `rank_bit`, applied by
        both partners in one peer-memory kernel each (csrc/peer.cu)."""
        self.transport.peer_barrier(self.engines)
        for eng, r in zip(self.engines, self.ranks):
            if (r & need) != need:
                continue
            partner = r ^ (1 << rank_bit)
            eng.peer_gate(self._peers[(r, partner)], not (r >> rank_bit) & 1, cmask, m)
        self.transport.peer_barrier(self.engines)
        self.peer_gate_count += 1

    def apply_op(self, gate, target: int, controls=()) -> "ShardedState":
        n = self.num_qubits
        qs = [int(target), *map(int, controls)]
        for q in qs:
            if not 0 <= q < n:
                raise IndexError(f"qubit {q} out of range for {n} qubits")
        if len(set(qs)) != len(qs):
            raise ValueError("control and target must differ")
        m = self._m8(gate)
        from .gates import is_phase

        kind = N.QS_OP_PHASE if is_phase(m) else N.QS_OP_PAIR
        lay = self.layout
        if kind == N.QS_OP_PHASE and not lay.is_local(target):
            # a diagonal gate is symmetric in its target/control bits: keep the
            # data in place and pick a local bit as the "target" if one exists
            local = [q for q in qs if lay.is_local(q)]
            if local:
                target = local[0]
                controls = [q for q in qs if q != target]
        if kind == N.QS_OP_PHASE and not any(lay.is_local(q) for q in qs):
            self._shard_phase([lay.pos[q] - lay.L for q in qs], m)
            return self
        if kind == N.QS_OP_PAIR and not lay.is_local(target) and self._global_pair_via_peer(lay.pos[target] - lay.L):
            cmask, need = self._control_masks(controls)
            self._peer_gate(lay.pos[target] - lay.L, cmask, need, m)
            return self
        if kind == N.QS_OP_PAIR or not any(lay.is_local(q) for q in [target, *controls]):
            self._ensure_local(target)
        t_phys = lay.pos[target]
        cmask, need_rank = 0, 0
        for c in controls:
            pc = lay.pos[c]
            if pc < lay.L:
                cmask |= 1 << pc
            else:
                need_rank |= 1 << (pc - lay.L)
        for eng, r in zip(self.engines, self.ranks):
            if (r & need_rank) == need_rank:
                eng.apply(kind, t_phys, cmask, m)
        return self

    def apply_gate(self, gate, target):
        return self.apply_op(gate, target)

    def apply_controlled_gate(self, gate, control, target):
        return self.apply_op(gate, target, (control,))

    def apply_controlled_controlled_gate(self, gate, c1, c2, target):
        return self.apply_op(gate, target, (c1, c2))

    def h(self, t):
        return self.apply_op(FIXED_GATES["h"], t)

    def x(self, t):
        return self.apply_op(FIXED_GATES["x"], t)

    def t(self, t):
        return self.apply_op(FIXED_GATES["t"], t)

    def cx(self, c, t):
        return self.apply_op(FIXED_GATES["x"], t, (c,))

    def cu1(self, c, t, theta):
        return self.apply_op(_u1(theta), t, (c,))

    def ccx(self, c1, c2, t):
        return self.apply_op(FIXED_GATES["x"], t, (c1, c2))

    def run(self, circuit, exact: bool = True) -> "ShardedState":
        """Apply a circuit: maximal runs of local ops go to each shard's fused
        planner in one call; global targets trigger a swap in between.
        exact=False: the shards' passes run in the inexact mode (reordered
        passes, combined diagonal runs; circuits.execute)."""
        from .circuits import Apply, ControlledApply, ControlledControlledApply

        pending: list = []

        def flush():
            if pending:
                for eng, r in zip(self.engines, self.ranks):
                    ops = [(k, t, cm, m) for (k, t, cm, m, need) in pending if (r & need) == need]
                    if ops:
                        if exact:
                            eng.apply_ops(ops)
                        else:
                            eng.apply_ops(ops, exact=False)
                pending.clear()

        for ins in circuit.instructions:
            if isinstance(ins, Apply):
                gate, target, controls = ins.gate, ins.target, ()
            elif isinstance(ins, ControlledApply):
                gate, target, controls = ins.gate, ins.target, (ins.control,)
            elif isinstance(ins, ControlledControlledApply):
                gate, target, controls = ins.gate, ins.target, (ins.control1, ins.control2)
            else:
                continue
            m = self._m8(gate)
            from .gates import is_phase

            kind = N.QS_OP_PHASE if is_phase(m) else N.QS_OP_PAIR
            lay = self.layout
            qs = [target, *controls]
            if kind == N.QS_OP_PHASE and not lay.is_local(target):
                local = [q for q in qs if lay.is_local(q)]
                if local:
                    target = local[0]
                    controls = tuple(q for q in qs if q != target)
            if kind == N.QS_OP_PHASE and not any(lay.is_local(q) for q in qs):
                flush()
                self._shard_phase([lay.pos[q] - lay.L for q in qs], m)
                continue
            if not lay.is_local(target):
                flush()
                if kind == N.QS_OP_PAIR and self._global_pair_via_peer(lay.pos[target] - lay.L):
                    cmask, need = self._control_masks(controls)
                    self._peer_gate(lay.pos[target] - lay.L, cmask, need, m)
                    continue
                self._ensure_local(target)  # moves qubits: masks after it
            cmask, need = self._control_masks(controls)
            pending.append((kind, lay.pos[target], cmask, m, need))
        flush()
        return self

    # ---- readout ---------------------------------------------------------------
    def canonicalize(self) -> "ShardedState":
        """Restore the identity qubit map (local swap kernels + exchanges)."""
        lay = self.layout
        for p in range(self.num_qubits):
            q = lay.at[p]
            if q == p:
                continue
            # bring logical qubit p (now at physical pp) to physical p
            pp = lay.pos[p]
            if p < lay.L and pp < lay.L:
                for eng in self.engines:
                    eng.swap_qubits(p, pp)
                lay.swap_physical(p, pp)
            elif p >= lay.L and pp >= lay.L:
                # swap two global positions through local L-1
                self._swap_global_via_local(p, pp)
            elif p < lay.L:  # target local, source global
                self._swap_local_global(p, pp)
            else:  # target global, source local
                self._swap_local_global(pp, p)
        return self

    def _swap_local_global(self, loc: int, glob: int) -> None:
        lay = self.layout
        s = lay.L - 1
        if loc != s:
            for eng in self.engines:
                eng.swap_qubits(loc, s)
            lay.swap_physical(loc, s)
        self._exchange(glob - lay.L)
        lay.swap_physical(glob, s)
        self.swaps += 1
        if loc != s:
            for eng in self.engines:
                eng.swap_qubits(loc, s)
            lay.swap_physical(loc, s)

    def _swap_global_via_local(self, g1: int, g2: int) -> None:
        self._swap_local_global(self.layout.L - 1, g1)
        self._swap_local_global(self.layout.L - 1, g2)
        self._swap_local_global(self.layout.L - 1, g1)

    def local_amplitudes(self):
        """{rank: amplitudes of its canonical slice} for the local engines."""
        self.canonicalize()
        return {r: eng.amplitudes() for eng, r in zip(self.engines, self.ranks)}

    def amplitudes(self) -> np.ndarray:
        """Full logical amplitude vector (virtual mode, or gathered over ranks)."""
        parts = self.local_amplitudes()
        if len(parts) == self.world:
            return np.concatenate([parts[r] for r in range(self.world)])
        return self._gather(parts, np.complex128 if self.double else np.complex64)

    def probabilities(self) -> np.ndarray:
        self.canonicalize()
        parts = {r: eng.probabilities() for eng, r in zip(self.engines, self.ranks)}
        if len(parts) == self.world:
            return np.concatenate([parts[r] for r in range(self.world)])
        return self._gather(parts, np.float64)

    def _gather(self, parts, dtype):
        import torch

        dist = self.transport.dist
        (r, arr), = parts.items()
        raw = np.ascontiguousarray(arr).view(np.uint8)
        t = torch.from_numpy(raw.copy())
        if dist.get_backend(self.transport.group) == "nccl":
            t = t.cuda()
        out = [torch.empty_like(t) for _ in range(self.world)]
        dist.all_gather(out, t, group=self.transport.group)
        return np.concatenate([o.cpu().numpy().view(dtype) for o in out])

    def sample_outcomes(self, samples: int, seed=None) -> np.ndarray:
        """Per-draw outcomes (logical basis indices), bit-exact with pairsim's
        sample on the full register (measure.py:76-85): the exact sequential
        CDF is chained across shards in index order."""
        from .errors import DegenerateStateError

        if samples < 1:
            raise ValueError("n_samples must be >= 1")
        self.canonicalize()
        rng = self.transport.common_seed_words(seed)
        starts, total = self.transport.cdf_chain(self.engines, self.ranks)
        if not total > 0.0:
            raise DegenerateStateError("all outcome probabilities are zero")
        L, dim = self.L, 1 << self.num_qubits
        outs = [eng.sample_shard(samples, rng, starts[r], total, r << L, dim, r == self.world - 1)
                for eng, r in zip(self.engines, self.ranks)]
        N.consume_draws(seed, samples)
        return self.transport.combine_max(outs)

    def measure(self, samples: int = 1000, seed=None) -> dict[int, int]:
        keys, counts = np.unique(self.sample_outcomes(samples, seed), return_counts=True)
        return dict(zip(keys.tolist(), counts.tolist()))  # Python ints, np.unique (sorted) order

    def measure_collapse(self, seed=None) -> int:
        """One draw, then the register becomes |outcome> (measure.py:88-99)."""
        m = int(self.sample_outcomes(1, seed)[0])
        self.reset(m)
        return m

    def norm_squared(self) -> float:
        vals = [eng.norm_squared() for eng in self.engines]
        if len(vals) == self.world:
            return float(sum(vals))
        return self.transport.allreduce_sum(vals)[0]

    def synchronize(self) -> None:
        for eng in self.engines:
            eng.synchronize()

    def close(self) -> None:
        """Unmap the partners' shards (behind a barrier: no rank may still be
        running a peer kernel on them), then free the local shards."""
        if self._peers:
            self.transport.peer_barrier(self.engines)
            by_rank = dict(zip(self.ranks, self.engines))
            for (r, _), ptr in self._peers.items():
                if hasattr(by_rank[r], "close_peer") and not isinstance(self.transport, LocalTransport):
                    by_rank[r].close_peer(ptr)
        self._peers = None
        for eng in self.engines:
            if hasattr(eng, "close"):
                eng.close()
        self.engines = []

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False
