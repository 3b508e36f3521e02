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

    def run(self, circuit) -> "MultiDeviceState":
        from .circuits import Apply, ControlledApply, ControlledControlledApply

        for ins in circuit.instructions:
            if isinstance(ins, Apply):
                self.apply_gate(ins.gate, ins.target)
            elif isinstance(ins, ControlledApply):
                self.apply_controlled_gate(ins.gate, ins.control, ins.target)
            elif isinstance(ins, ControlledControlledApply):
                self.apply_controlled_controlled_gate(ins.gate, ins.control1, ins.control2, ins.target)
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
        return {int(k): int(c) for k, c in zip(keys, counts)}

    def __repr__(self) -> str:
        return f"MultiDeviceState(num_qubits={self.num_qubits}, devices={self.devices})"
