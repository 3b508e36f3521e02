"""One process, several GPUs: the C-ABI sharded register (qs_create_sharded,
include/qsb200.h; csrc/sharded.cu) behind the QCGPU-style State API.

    reg = MultiDeviceState(36, devices=[0, 1, 2, 3, 4, 5, 6, 7])
    reg.h(35); reg.cx(35, 0); reg.probabilities(); reg.measure(1000)

The register of n qubits is split over len(devices) = 2^g shards on its top
g qubits; global-qubit gates move data with NCCL send/recv
between the devices (one communicator per device, ncclCommInitAll) or over
peer memory.  No torch in this path: ctypes straight into libqsb200.
Devices may repeat (several shards on one GPU), which is how the one-GPU
tests exercise the same code.  The multi-PROCESS form (one rank per GPU under
torchrun) is paper_1805_00988_b200.sharded.ShardedState.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native as N
from .gates import FIXED_GATES, m8, u1 as _u1


class _Shard:
    """One shard's qs_state as the object fusion.run drives (State's fused-pass
    entry points on a borrowed handle; the register owns the shard)."""

    def __init__(self, reg: "MultiDeviceState", rank: int, num_qubits: int):
        ptr = ctypes.c_void_p()
        N.check(N.lib().qs_sharded_shard(reg.handle, int(rank), ctypes.byref(ptr)))
        self.handle = ptr
        self.num_qubits = num_qubits
        self.is_double = False

    def apply_fused(self, tile_qubits, ops, combine: bool = False):
        from .state import State

        return State.apply_fused(self, tile_qubits, ops, combine)


class MultiDeviceState:
    def __init__(self, num_qubits: int, devices, memory_budget: int | None = None,
                 peer_gates: bool | None = None, exchange: str | None = None):
        devs = [int(d) for d in devices]
        arr = (ctypes.c_int * len(devs))(*devs)
        h = ctypes.c_void_p()
        N.check(N.lib().qs_create_sharded(int(num_qubits), len(devs), arr, int(memory_budget or 0),
                                          ctypes.byref(h)))
        self._h = h
        self.num_qubits = int(num_qubits)
        self.devices = devs
        if peer_gates is not None or exchange is not None:
            self.set_mode(peer_gates, exchange)

    # ---- lifecycle ------------------------------------------------------------
    @property
    def handle(self):
        if self._h is None or not self._h.value:
            raise ValueError("register is closed")
        return self._h

    def close(self) -> None:
        if self._h is not None and self._h.value:
            N.lib().qs_sharded_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def set_mode(self, peer_gates: bool | None = None, exchange: str | None = None) -> None:
        ex = {None: 0, "nccl": N.QS_EXCHANGE_NCCL, "p2p": N.QS_EXCHANGE_P2P, "peer": N.QS_EXCHANGE_P2P}[exchange]
        N.check(N.lib().qs_sharded_set_mode(self.handle, -1 if peer_gates is None else int(bool(peer_gates)), ex))

    def stats(self) -> dict:
        sw, pg, ex = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_int()
        N.check(N.lib().qs_sharded_stats(self.handle, ctypes.byref(sw), ctypes.byref(pg), ctypes.byref(ex)))
        return {"swaps": sw.value, "peer_gates": pg.value,
                "exchange": {N.QS_EXCHANGE_NCCL: "nccl", N.QS_EXCHANGE_P2P: "p2p"}.get(ex.value, "?")}

    @property
    def shard_qubits(self) -> int:
        L = ctypes.c_int()
        N.check(N.lib().qs_sharded_info(self.handle, None, None, ctypes.byref(L)))
        return L.value

    # ---- gates (pairsim kernel.py:108-165 semantics) --------------------------
    def reset(self, basis: int = 0) -> "MultiDeviceState":
        N.check(N.lib().qs_sharded_reset(self.handle, int(basis)))
        return self

    def apply_gate(self, gate, target: int):
        N.check(N.lib().qs_sharded_apply_gate(self.handle, int(target), N.f32ptr(m8(gate))))
        return self

    def apply_controlled_gate(self, gate, control: int, target: int):
        N.check(N.lib().qs_sharded_apply_controlled_gate(self.handle, int(control), int(target), N.f32ptr(m8(gate))))
        return self

    def apply_controlled_controlled_gate(self, gate, c1: int, c2: int, target: int):
        N.check(N.lib().qs_sharded_apply_controlled_controlled_gate(self.handle, int(c1), int(c2), int(target),
                                                                    N.f32ptr(m8(gate))))
        return self

    def h(self, t):
        return self.apply_gate(FIXED_GATES["h"], t)

    def x(self, t):
        return self.apply_gate(FIXED_GATES["x"], t)

    def y(self, t):
        return self.apply_gate(FIXED_GATES["y"], t)

    def z(self, t):
        return self.apply_gate(FIXED_GATES["z"], t)

    def s(self, t):
        return self.apply_gate(FIXED_GATES["s"], t)

    def t(self, t):
        return self.apply_gate(FIXED_GATES["t"], t)

    def u1(self, t, theta: float):
        return self.apply_gate(_u1(theta), t)

    def cx(self, control, target):
        return self.apply_controlled_gate(FIXED_GATES["x"], control, target)

    def cu1(self, control, target, theta: float):
        return self.apply_controlled_gate(_u1(theta), control, target)

    def ccx(self, c1, c2, target):
        return self.apply_controlled_controlled_gate(FIXED_GATES["x"], c1, c2, target)

    def qubit_map(self) -> list[int]:
        """pos[logical qubit] = physical position (>= shard_qubits: global)."""
        arr = (ctypes.c_int32 * self.num_qubits)()
        N.check(N.lib().qs_sharded_qubit_map(self.handle, arr))
        return list(arr)

    def run(self, circuit, fuse: bool = True, exact: bool = True) -> "MultiDeviceState":
        """Apply a circuit.  fuse=True: maximal runs of local ops run as fused
        passes on every shard (the single-device planner and kernels, through
        each shard's qs_state); a pair gate on a global qubit (qubit swap or
        peer gate) and a diagonal gate on global-only bits go through the C
        ABI in between.  exact=False as in circuits.execute."""
        from . import fusion
        from .circuits import Apply, ControlledApply, ControlledControlledApply
        from .gates import is_phase

        def split(ins):
            if isinstance(ins, Apply):
                return ins.gate, ins.target, ()
            if isinstance(ins, ControlledApply):
                return ins.gate, ins.target, (ins.control,)
            if isinstance(ins, ControlledControlledApply):
                return ins.gate, ins.target, (ins.control1, ins.control2)
            return None

        def one(gate, target, controls):
            if not controls:
                self.apply_gate(gate, target)
            elif len(controls) == 1:
                self.apply_controlled_gate(gate, controls[0], target)
            else:
                self.apply_controlled_controlled_gate(gate, controls[0], controls[1], target)

        if not fuse:
            for ins in circuit.instructions:
                g = split(ins)
                if g is not None:
                    one(*g)
            return self
        L = self.shard_qubits
        shards = [_Shard(self, r, L) for r in range(len(self.devices))]
        pending: list = []

        def flush():
            for r, sh in enumerate(shards):
                ops = [(k, t, cm, m) for (k, t, cm, m, need) in pending if (r & need) == need]
                if ops:
                    fusion.run(sh, fusion.plan(L, ops, reorder=not exact), combine=not exact)
            pending.clear()

        pos = self.qubit_map()
        for ins in circuit.instructions:
            g = split(ins)
            if g is None:
                continue
            gate, target, controls = g
            m = m8(gate)
            kind = N.QS_OP_PHASE if is_phase(m) else N.QS_OP_PAIR
            qs = [target, *controls]
            if kind == N.QS_OP_PHASE and pos[target] >= L:
                local = [q for q in qs if pos[q] < L]
                if local:
                    target, controls = local[0], tuple(q for q in qs if q != local[0])
            if pos[target] >= L:  # global pair target, or a diagonal gate on global-only bits
                flush()
                one(gate, *g[1:])
                pos = self.qubit_map()
                continue
            cmask, need = 0, 0
            for c in controls:
                if pos[c] < L:
                    cmask |= 1 << pos[c]
                else:
                    need |= 1 << (pos[c] - L)
            pending.append((kind, pos[target], cmask, m, need))
        flush()
        return self

    def flush(self) -> None:
        N.check(N.lib().qs_sharded_synchronize(self.handle))

    # ---- readout ----------------------------------------------------------------
    @property
    def dim(self) -> int:
        return 1 << self.num_qubits

    def amplitudes(self, offset: int = 0, count: int | None = None) -> np.ndarray:
        count = self.dim - offset if count is None else count
        out = np.empty(count, np.complex64)
        N.check(N.lib().qs_sharded_get_amplitudes(self.handle, int(offset), int(count), out.ctypes.data))
        return out

    def set_amplitudes(self, values, offset: int = 0) -> None:
        arr = np.ascontiguousarray(values, dtype=np.complex64)
        N.check(N.lib().qs_sharded_set_amplitudes(self.handle, int(offset), arr.size, arr.ctypes.data))

    def probabilities(self, offset: int = 0, count: int | None = None) -> np.ndarray:
        count = self.dim - offset if count is None else count
        out = np.empty(count, np.float64)
        N.check(N.lib().qs_sharded_probabilities(self.handle, int(offset), int(count), out.ctypes.data))
        return out

    def norm_squared(self) -> float:
        v = ctypes.c_double()
        N.check(N.lib().qs_sharded_norm_squared(self.handle, ctypes.byref(v)))
        return v.value

    def sample_outcomes(self, samples: int, seed=None) -> np.ndarray:
        """Per-draw outcomes, bit-exact with pairsim.measure.sample on the whole register."""
        if samples < 1:
            raise ValueError("n_samples must be >= 1")
        out = np.empty(int(samples), np.int64)
        rng = N.pcg_from_seed(seed)
        N.check(N.lib().qs_sharded_sample(self.handle, ctypes.byref(rng), int(samples), out.ctypes.data))
        N.consume_draws(seed, samples)
        return out

    def measure(self, samples: int = 1000, seed=None) -> dict[int, int]:
        keys, counts = np.unique(self.sample_outcomes(samples, seed), return_counts=True)
        return dict(zip(keys.tolist(), counts.tolist()))  # Python ints, np.unique (sorted) order

    def __repr__(self) -> str:
        return f"MultiDeviceState(num_qubits={self.num_qubits}, devices={self.devices})"
