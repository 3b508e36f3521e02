"""QCGPU-style register object: ``State(n)`` living in B200 HBM.

API (north_star):
    s = State(n)                        # |0...0>, complex64 in HBM
    s = State(n, precision="double")    # complex128 (pairsim Precision.DOUBLE)
    s.apply_gate(gate, target)
    s.apply_controlled_gate(gate, control, target)
    s.apply_controlled_controlled_gate(gate, c1, c2, target)
    s.h(t) s.x(t) s.y(t) s.z(t) s.s(t) s.t(t) s.u1(t, theta)
    s.cx(c, t) s.cu1(c, t, theta) s.ccx(c1, c2, t)  # control(s) first
    s.amplitudes() -> complex64 (complex128) ndarray
    s.probabilities() -> float64 ndarray
    s.measure(samples=1000, seed=None) -> {basis_index: count}
    s.flush(); s.backend.queue.finish()  # device barrier

Gate semantics are the reference's pair sweep (pkg/src/pairsim/kernel.py:108-165);
every call is one asynchronous launch on the state's CUDA stream.
"""

from __future__ import annotations

import ctypes
import math

import numpy as np

from . import _native as N
from .gates import FIXED_GATES, Gate, entries_ptr, u1 as _u1


class _Queue:
    def __init__(self, state: "State"):
        self._state = state

    def finish(self) -> None:
        self._state.flush()


class Graph:
    """A recorded gate sequence (CUDA graph) of one State; replay() runs it
    again as a single graph launch (qs_graph_launch)."""

    def __init__(self, state: "State", handle: ctypes.c_void_p):
        self._state = state
        self._h = handle

    def replay(self, times: int = 1) -> "State":
        for _ in range(int(times)):
            N.check(N.lib().qs_graph_launch(self._state.handle, self._h))
        return self._state

    def close(self) -> None:
        if self._h is not None and self._h.value:
            N.lib().qs_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _Recording:
    def __init__(self, state: "State"):
        self._state = state
        self.graph: Graph | None = None

    def __enter__(self):
        import gc

        # no garbage-collected State may free its buffer mid-recording; gc is
        # turned off only once the capture has started (a failed begin leaves
        # the collector as it was)
        h = self._state.handle
        self._gc = gc.isenabled()
        N.check(N.lib().qs_begin_capture(h))
        gc.disable()
        return self

    def __exit__(self, exc_type, exc, tb):
        import gc

        h = ctypes.c_void_p()
        rc = N.lib().qs_end_capture(self._state.handle, ctypes.byref(h))
        if self._gc:
            gc.enable()
        if exc_type is None:
            N.check(rc)
            self.graph = Graph(self._state, h)
        elif h.value:
            N.lib().qs_graph_destroy(h)
        return False


class _Backend:
    """``state.backend.queue.finish()`` compatibility."""

    def __init__(self, state: "State"):
        self.queue = _Queue(state)


def _precision_code(precision) -> int:
    """'single' / 'double', numpy complex dtypes, or pairsim Precision members."""
    v = getattr(precision, "value", precision)
    if isinstance(v, str) and v.lower() in ("single", "complex64", "c64"):
        return N.QS_SINGLE
    if isinstance(v, str) and v.lower() in ("double", "complex128", "c128"):
        return N.QS_DOUBLE
    try:
        dt = np.dtype(v)
    except TypeError:
        dt = None
    if dt == np.complex64:
        return N.QS_SINGLE
    if dt == np.complex128:
        return N.QS_DOUBLE
    raise ValueError(f"unsupported precision {precision!r}")


class State:
    def __init__(self, num_qubits: int, device: int = 0, memory_budget: int | None = None,
                 precision="single", _init: bool = True):
        if not isinstance(num_qubits, (int, np.integer)):
            raise TypeError("num_qubits must be an integer")
        if num_qubits < 1:
            raise ValueError("num_qubits must be >= 1")
        prec = _precision_code(precision)
        self._h = ctypes.c_void_p()
        # _init=False: contents undefined until the first fused pass writes its
        # start state (execute(..., initial_basis=b) right after; qs_create_uninit)
        create = N.lib().qs_create_ex if _init else N.lib().qs_create_uninit
        N.check(create(int(num_qubits), int(device), int(memory_budget or 0), prec, ctypes.byref(self._h)))
        self.num_qubits = int(num_qubits)
        self.device = int(device)
        self.is_double = prec == N.QS_DOUBLE
        self.dtype = np.dtype(np.complex128 if self.is_double else np.complex64)
        self.backend = _Backend(self)

    # -- lifecycle ------------------------------------------------------------
    def close(self) -> None:
        if getattr(self, "_h", None) and self._h.value:
            N.lib().qs_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    @property
    def handle(self) -> ctypes.c_void_p:
        if not self._h.value:
            raise ValueError("state has been closed")
        return self._h

    @property
    def dim(self) -> int:
        return 1 << self.num_qubits

    def device_pointer(self) -> int:
        p = ctypes.c_void_p()
        N.check(N.lib().qs_device_pointer(self.handle, ctypes.byref(p)))
        return p.value

    def stream(self) -> int:
        p = ctypes.c_void_p()
        N.check(N.lib().qs_stream(self.handle, ctypes.byref(p)))
        return p.value or 0

    def flush(self) -> None:
        N.check(N.lib().qs_synchronize(self.handle))

    def reset(self, basis: int = 0) -> "State":
        N.check(N.lib().qs_reset(self.handle, int(basis)))
        return self

    # -- gates ----------------------------------------------------------------
    # Gate entries are rounded to the register's precision first
    # (kernel.py:118-119): float32 entry points for complex64, fp64 for complex128.
    def _m(self, gate):
        m, ptr = entries_ptr(gate, self.is_double)
        return ptr, m

    def apply_gate(self, gate, target: int) -> "State":
        mp, _keep = self._m(gate)
        L = N.lib()
        fn = L.qs_apply_gate_f64 if self.is_double else L.qs_apply_gate
        N.check(fn(self.handle, int(target), mp))
        return self

    def apply_controlled_gate(self, gate, control: int, target: int) -> "State":
        mp, _keep = self._m(gate)
        L = N.lib()
        fn = L.qs_apply_controlled_gate_f64 if self.is_double else L.qs_apply_controlled_gate
        N.check(fn(self.handle, int(control), int(target), mp))
        return self

    def apply_controlled_controlled_gate(self, gate, control1: int, control2: int, target: int) -> "State":
        mp, _keep = self._m(gate)
        L = N.lib()
        fn = (L.qs_apply_controlled_controlled_gate_f64 if self.is_double
              else L.qs_apply_controlled_controlled_gate)
        N.check(fn(self.handle, int(control1), int(control2), int(target), mp))
        return self

    def apply_fused(self, tile_qubits, ops: np.ndarray, combine: bool = False,
                    from_basis: int | None = None, chunk_sums: bool = False) -> "State":
        """One fused HBM pass (see fusion.py for the planner).  `ops` is an
        OP_DTYPE (float32 entries) or OP64_DTYPE (fp64 entries) record array.
        combine=True (not bit-exact, QS_FUSED_COMBINE_PHASES): runs of
        unit-modulus diagonal ops become one product per amplitude.
        from_basis=b: reset to |b> first, folded into the pass (its tiles are
        written as |b> instead of loaded: qs_apply_fused_from_basis).
        chunk_sums=True: the pass also leaves the sampler's chunk sums (after
        sample_prepare; QS_FUSED_CHUNK_SUMS)."""
        tq = np.ascontiguousarray(np.asarray(tile_qubits, dtype=np.int32))
        wide = np.asarray(ops).dtype == N.OP64_DTYPE
        ops = np.ascontiguousarray(ops, dtype=N.OP64_DTYPE if wide else N.OP_DTYPE)
        L = N.lib()
        tp = tq.ctypes.data_as(ctypes.POINTER(ctypes.c_int32))
        flags = (N.QS_FUSED_COMBINE_PHASES if combine else 0) | (N.QS_FUSED_CHUNK_SUMS if chunk_sums else 0)
        if from_basis is not None:
            if wide:
                self.reset(int(from_basis))
            else:
                N.check(L.qs_apply_fused_from_basis(self.handle, tp, int(tq.size), ops.ctypes.data, int(ops.size),
                                                    flags, int(from_basis)))
                return self
        if wide:
            N.check(L.qs_apply_fused_f64(self.handle, tp, int(tq.size), ops.ctypes.data, int(ops.size)))
        elif flags:
            N.check(L.qs_apply_fused_ex(self.handle, tp, int(tq.size), ops.ctypes.data, int(ops.size), flags))
        else:
            N.check(L.qs_apply_fused(self.handle, tp, int(tq.size), ops.ctypes.data, int(ops.size)))
        return self

    def record(self) -> "_Recording":
        """Record the gate launches of a block into a CUDA graph instead of running them:

            with st.record() as rec:
                execute(circuit, st)
            rec.graph.replay(100)

        Only asynchronous calls (gates, fused passes, reset, uploads) may be
        recorded; fused passes whose compiled program is not loaded yet are
        recorded on the interpreter kernel (same bits)."""
        return _Recording(self)

    def swap_qubits(self, q1: int, q2: int) -> "State":
        N.check(N.lib().qs_swap_qubits(self.handle, int(q1), int(q2)))
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

    def cz(self, control, target):
        return self.apply_controlled_gate(FIXED_GATES["z"], control, target)

    def cu1(self, control, target, theta: float):
        return self.apply_controlled_gate(_u1(theta), control, target)

    def ccx(self, control1, control2, target):
        return self.apply_controlled_controlled_gate(FIXED_GATES["x"], control1, control2, target)

    # -- readout ----------------------------------------------------------------
    def amplitudes(self, offset: int = 0, count: int | None = None) -> np.ndarray:
        count = self.dim - offset if count is None else count
        out = np.empty(count, dtype=self.dtype)
        N.check(N.lib().qs_get_amplitudes(self.handle, int(offset), int(count), out.ctypes.data))
        return out

    def set_amplitudes(self, values, offset: int = 0) -> "State":
        v = np.ascontiguousarray(np.asarray(values), dtype=self.dtype)
        N.check(N.lib().qs_set_amplitudes(self.handle, int(offset), int(v.size), v.ctypes.data))
        return self

    def upload_async(self, host_ptr: int, count: int | None = None, offset: int = 0) -> "State":
        """Enqueue a host->device copy from a (pinned) buffer address; the buffer
        must stay valid until flush()."""
        count = self.dim - offset if count is None else count
        N.check(N.lib().qs_set_amplitudes_async(self.handle, int(offset), int(count), int(host_ptr)))
        return self

    def download_async(self, host_ptr: int, count: int | None = None, offset: int = 0) -> "State":
        """Enqueue a device->host copy into a (pinned) buffer address."""
        count = self.dim - offset if count is None else count
        N.check(N.lib().qs_get_amplitudes_async(self.handle, int(offset), int(count), int(host_ptr)))
        return self

    def amplitude(self, index: int) -> complex:
        if not 0 <= index < self.dim:
            raise IndexError(f"basis index {index} out of range [0, {self.dim})")
        return complex(self.amplitudes(index, 1)[0])

    def probabilities(self, offset: int = 0, count: int | None = None, out: np.ndarray | None = None) -> np.ndarray:
        """fp64 |a|^2 (measure.py:29-34).  `out`: a float64 array to fill (e.g.
        _native.pinned_empty(2**n): page-locked, filled by DMA with no staging
        copy), else a fresh array."""
        count = self.dim - offset if count is None else count
        if out is None:
            out = np.empty(count, dtype=np.float64)
        elif out.dtype != np.float64 or out.size != count or not out.flags.c_contiguous:
            raise ValueError("out must be a contiguous float64 array of `count` elements")
        N.check(N.lib().qs_probabilities(self.handle, int(offset), int(count), out.ctypes.data))
        return out

    def norm_squared(self) -> float:
        v = ctypes.c_double()
        N.check(N.lib().qs_norm_squared(self.handle, ctypes.byref(v)))
        return v.value

    def sample_outcomes(self, samples: int, seed=None, sums_ready: bool = False) -> np.ndarray:
        """Per-draw outcomes, bit-exact with pairsim.measure.sample for the same seed.
        sums_ready: the last fused pass accumulated the sampler's chunk sums
        (sample_prepare + apply_fused(chunk_sums=True)); a shortcut only."""
        if samples < 1:
            raise ValueError("n_samples must be >= 1")
        out = np.empty(int(samples), dtype=np.int64)
        rng = N.pcg_from_seed(seed)
        N.check(N.lib().qs_sample_ex(self.handle, ctypes.byref(rng), int(samples), out.ctypes.data,
                                     N.QS_SAMPLE_SUMS_READY if sums_ready else 0))
        N.consume_draws(seed, samples)
        return out

    def sample_prepare(self, samples: int) -> "State":
        """Lay out the sampler's scratch for `samples` draws so the next fused
        pass (apply_fused(chunk_sums=True)) can leave the chunk sums."""
        N.check(N.lib().qs_sample_prepare(self.handle, int(samples)))
        return self

    def cdf_extend(self, start: float) -> float:
        """Exact sequential cumsum of this register's probabilities continued from `start`."""
        end = ctypes.c_double()
        N.check(N.lib().qs_cdf_extend(self.handle, float(start), ctypes.byref(end)))
        return end.value

    def sample_shard(self, samples: int, rng: "N.qs_pcg64", start: float, total: float,
                     base: int, global_dim: int, is_last: bool) -> np.ndarray:
        """Draws of a global register of which this is the slice [base, base + 2^n):
        global outcomes for draws landing here, -1 elsewhere (qs_sample_shard)."""
        out = np.empty(int(samples), dtype=np.int64)
        N.check(N.lib().qs_sample_shard(self.handle, ctypes.byref(rng), int(samples), float(start),
                                        float(total), int(base), int(global_dim), int(bool(is_last)),
                                        out.ctypes.data))
        return out

    def measure(self, samples: int = 1000, seed=None) -> dict[int, int]:
        """Non-destructive sampling: {basis index: count}."""
        keys, counts = np.unique(self.sample_outcomes(samples, seed), return_counts=True)
        return dict(zip(keys.tolist(), counts.tolist()))  # Python ints, np.unique (sorted) order

    def measure_bitstrings(self, samples: int = 1000, seed=None) -> dict[str, int]:
        """Same draws keyed by the n-bit string (qubit n-1 first)."""
        return {format(k, f"0{self.num_qubits}b"): c for k, c in self.measure(samples, seed).items()}

    def measure_collapse(self, seed=None) -> int:
        out = ctypes.c_int64()
        rng = N.pcg_from_seed(seed)
        N.check(N.lib().qs_measure_collapse(self.handle, ctypes.byref(rng), ctypes.byref(out)))
        N.consume_draws(seed, 1)
        return int(out.value)

    # ---- checkpoint / resume: the amplitudes as a .npy file -----
    _CHUNK = 1 << 26  # amplitudes per host transfer (512 MiB of complex64)

    def save(self, path) -> None:
        """Write the register to `path` as a .npy array (complex64 or
        complex128), streamed in chunks (no full host copy)."""
        mm = np.lib.format.open_memmap(str(path), mode="w+", dtype=self.dtype, shape=(self.dim,))
        try:
            for off in range(0, self.dim, self._CHUNK):
                cnt = min(self._CHUNK, self.dim - off)
                mm[off: off + cnt] = self.amplitudes(off, cnt)
            mm.flush()
        finally:
            del mm

    @classmethod
    def load(cls, path, device: int = 0, memory_budget: int | None = None) -> "State":
        """A new register holding the amplitudes saved by `save` (or any 1-D
        complex64 / complex128 .npy array of length 2^n)."""
        arr = np.load(str(path), mmap_mode="r")
        n = int(arr.shape[0]).bit_length() - 1
        if arr.ndim != 1 or arr.shape[0] != 1 << n or arr.dtype not in (np.complex64, np.complex128):
            raise ValueError("expected a 1-D complex64/complex128 array of length 2^n")
        st = cls(n, device=device, memory_budget=memory_budget, precision=arr.dtype)
        for off in range(0, arr.shape[0], cls._CHUNK):
            cnt = min(cls._CHUNK, arr.shape[0] - off)
            st.set_amplitudes(np.ascontiguousarray(arr[off: off + cnt]), offset=off)
        return st

    def __repr__(self) -> str:
        prec = ", precision='double'" if self.is_double else ""
        return f"State(num_qubits={self.num_qubits}, device={self.device}{prec})"
