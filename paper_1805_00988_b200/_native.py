"""ctypes binding of libqsb200.so (include/qsb200.h).

There is no CPU fallback: if the library is missing, or no CUDA device is
visible, every operation raises.  The library is built in-tree by
``python -m paper_1805_00988_b200.build`` (or __graft_entry__.build()).
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

import numpy as np

from .errors import CapacityError, DegenerateStateError, DeviceError

LIB_PATH = Path(__file__).resolve().parent / "libqsb200.so"
if os.environ.get("QSB_LIB"):  # A/B experiments with an alternative in-tree build
    LIB_PATH = Path(os.environ["QSB_LIB"]).resolve()

QS_OK, QS_ERR_INDEX, QS_ERR_VALUE, QS_ERR_CAPACITY, QS_ERR_DEGENERATE, QS_ERR_CUDA, QS_ERR_NULL = range(7)
QS_OP_PAIR, QS_OP_PHASE = 0, 1
QS_SINGLE, QS_DOUBLE = 0, 1

# Every symbol include/qsb200.h declares (checked by tests/test_native_abi.py).
EXPORTS = (
    "qs_abi_version", "qs_last_error", "qs_device_count", "qs_release_cached", "qs_host_alloc", "qs_host_free",
    "qs_create", "qs_create_ex", "qs_create_uninit",
    "qs_precision", "qs_destroy",
    "qs_num_qubits", "qs_device", "qs_device_pointer", "qs_stream", "qs_reset",
    "qs_synchronize", "qs_apply_gate", "qs_apply_controlled_gate",
    "qs_apply_controlled_controlled_gate", "qs_apply_gate_f64", "qs_apply_controlled_gate_f64",
    "qs_apply_controlled_controlled_gate_f64", "qs_apply_fused", "qs_apply_fused_ex", "qs_apply_fused_from_basis", "qs_apply_fused_f64", "qs_swap_qubits",
    "qs_get_amplitudes", "qs_set_amplitudes", "qs_get_amplitudes_async", "qs_set_amplitudes_async",
    "qs_probabilities", "qs_norm_squared",
    "qs_sample", "qs_sample_prepare", "qs_sample_ex", "qs_measure_collapse", "qs_cdf_extend", "qs_sample_shard",
    "qs_ipc_handle", "qs_ipc_open", "qs_ipc_close", "qs_apply_gate_peer", "qs_apply_gate_peer_f64", "qs_swap_peer", "qs_jit_sync", "qs_jit_stats",
    "qs_jit_shutdown", "qs_begin_capture", "qs_end_capture", "qs_graph_launch", "qs_graph_destroy",
    "qs_create_sharded", "qs_sharded_destroy", "qs_sharded_info", "qs_sharded_shard", "qs_sharded_set_mode",
    "qs_sharded_stats", "qs_sharded_reset", "qs_sharded_apply_gate", "qs_sharded_apply_controlled_gate",
    "qs_sharded_apply_controlled_controlled_gate", "qs_sharded_synchronize", "qs_sharded_get_amplitudes",
    "qs_sharded_set_amplitudes", "qs_sharded_probabilities", "qs_sharded_norm_squared", "qs_sharded_sample",
    "qs_sharded_qubit_map", "qs_sharded_localize",
)
QS_EXCHANGE_NCCL, QS_EXCHANGE_P2P = 1, 2
QS_FUSED_COMBINE_PHASES = 1
QS_FUSED_CHUNK_SUMS = 2
QS_SAMPLE_SUMS_READY = 1


class qs_pcg64(ctypes.Structure):
    _fields_ = [("state_hi", ctypes.c_uint64), ("state_lo", ctypes.c_uint64),
                ("inc_hi", ctypes.c_uint64), ("inc_lo", ctypes.c_uint64)]


class qs_op(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("target", ctypes.c_int32),
                ("ctrl_mask", ctypes.c_uint64), ("m", ctypes.c_float * 8)]


class qs_op64(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("target", ctypes.c_int32),
                ("ctrl_mask", ctypes.c_uint64), ("m", ctypes.c_double * 8)]


OP_DTYPE = np.dtype([("kind", np.int32), ("target", np.int32), ("ctrl_mask", np.uint64),
                     ("m", np.float32, 8)])
OP64_DTYPE = np.dtype([("kind", np.int32), ("target", np.int32), ("ctrl_mask", np.uint64),
                       ("m", np.float64, 8)])
assert OP_DTYPE.itemsize == ctypes.sizeof(qs_op)
assert OP64_DTYPE.itemsize == ctypes.sizeof(qs_op64)

_lib = None


def _declare(L):
    vp = ctypes.c_void_p
    i32, u64, i64 = ctypes.c_int, ctypes.c_uint64, ctypes.c_int64
    f32p = ctypes.POINTER(ctypes.c_float)
    f64p = ctypes.POINTER(ctypes.c_double)
    sig = {
        "qs_abi_version": ([], i32),
        "qs_last_error": ([], ctypes.c_char_p),
        "qs_device_count": ([ctypes.POINTER(i32)], i32),
        "qs_release_cached": ([i32], i32),
        "qs_host_alloc": ([u64, ctypes.POINTER(vp)], i32),
        "qs_host_free": ([vp], i32),
        "qs_create": ([i32, i32, u64, ctypes.POINTER(vp)], i32),
        "qs_create_ex": ([i32, i32, u64, i32, ctypes.POINTER(vp)], i32),
        "qs_create_uninit": ([i32, i32, u64, i32, ctypes.POINTER(vp)], i32),
        "qs_precision": ([vp, ctypes.POINTER(i32)], i32),
        "qs_destroy": ([vp], i32),
        "qs_num_qubits": ([vp, ctypes.POINTER(i32)], i32),
        "qs_device": ([vp, ctypes.POINTER(i32)], i32),
        "qs_device_pointer": ([vp, ctypes.POINTER(vp)], i32),
        "qs_stream": ([vp, ctypes.POINTER(vp)], i32),
        "qs_reset": ([vp, u64], i32),
        "qs_synchronize": ([vp], i32),
        "qs_apply_gate": ([vp, i32, f32p], i32),
        "qs_apply_controlled_gate": ([vp, i32, i32, f32p], i32),
        "qs_apply_controlled_controlled_gate": ([vp, i32, i32, i32, f32p], i32),
        "qs_apply_gate_f64": ([vp, i32, f64p], i32),
        "qs_apply_controlled_gate_f64": ([vp, i32, i32, f64p], i32),
        "qs_apply_controlled_controlled_gate_f64": ([vp, i32, i32, i32, f64p], i32),
        "qs_apply_fused": ([vp, ctypes.POINTER(ctypes.c_int32), i32, vp, i32], i32),
        "qs_apply_fused_f64": ([vp, ctypes.POINTER(ctypes.c_int32), i32, vp, i32], i32),
        "qs_apply_fused_ex": ([vp, ctypes.POINTER(ctypes.c_int32), i32, vp, i32, i32], i32),
        "qs_apply_fused_from_basis": ([vp, ctypes.POINTER(ctypes.c_int32), i32, vp, i32, i32, ctypes.c_uint64], i32),
        "qs_swap_qubits": ([vp, i32, i32], i32),
        "qs_get_amplitudes": ([vp, u64, u64, vp], i32),
        "qs_set_amplitudes": ([vp, u64, u64, vp], i32),
        "qs_get_amplitudes_async": ([vp, u64, u64, vp], i32),
        "qs_set_amplitudes_async": ([vp, u64, u64, vp], i32),
        "qs_probabilities": ([vp, u64, u64, vp], i32),
        "qs_norm_squared": ([vp, ctypes.POINTER(ctypes.c_double)], i32),
        "qs_sample": ([vp, ctypes.POINTER(qs_pcg64), i64, vp], i32),
        "qs_sample_prepare": ([vp, i64], i32),
        "qs_sample_ex": ([vp, ctypes.POINTER(qs_pcg64), i64, vp, i32], i32),
        "qs_measure_collapse": ([vp, ctypes.POINTER(qs_pcg64), ctypes.POINTER(i64)], i32),
        "qs_cdf_extend": ([vp, ctypes.c_double, ctypes.POINTER(ctypes.c_double)], i32),
        "qs_sample_shard": ([vp, ctypes.POINTER(qs_pcg64), i64, ctypes.c_double, ctypes.c_double,
                             u64, u64, i32, vp], i32),
        "qs_ipc_handle": ([vp, vp], i32),
        "qs_ipc_open": ([i32, vp, ctypes.POINTER(vp)], i32),
        "qs_ipc_close": ([i32, vp], i32),
        "qs_apply_gate_peer": ([vp, vp, i32, u64, f32p], i32),
        "qs_swap_peer": ([vp, vp, u64, u64, u64], i32),
        "qs_apply_gate_peer_f64": ([vp, vp, i32, u64, f64p], i32),
        "qs_create_sharded": ([i32, i32, ctypes.POINTER(i32), u64, ctypes.POINTER(vp)], i32),
        "qs_sharded_destroy": ([vp], i32),
        "qs_sharded_info": ([vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32)], i32),
        "qs_sharded_shard": ([vp, i32, ctypes.POINTER(vp)], i32),
        "qs_sharded_set_mode": ([vp, i32, i32], i32),
        "qs_sharded_stats": ([vp, ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(i32)], i32),
        "qs_sharded_reset": ([vp, u64], i32),
        "qs_sharded_apply_gate": ([vp, i32, f32p], i32),
        "qs_sharded_apply_controlled_gate": ([vp, i32, i32, f32p], i32),
        "qs_sharded_apply_controlled_controlled_gate": ([vp, i32, i32, i32, f32p], i32),
        "qs_sharded_synchronize": ([vp], i32),
        "qs_sharded_get_amplitudes": ([vp, u64, u64, vp], i32),
        "qs_sharded_set_amplitudes": ([vp, u64, u64, vp], i32),
        "qs_sharded_probabilities": ([vp, u64, u64, vp], i32),
        "qs_sharded_norm_squared": ([vp, ctypes.POINTER(ctypes.c_double)], i32),
        "qs_sharded_sample": ([vp, ctypes.POINTER(qs_pcg64), i64, vp], i32),
        "qs_sharded_qubit_map": ([vp, ctypes.POINTER(ctypes.c_int32)], i32),
        "qs_sharded_localize": ([vp, i32], i32),
        "qs_jit_sync": ([i32], i32),
        "qs_jit_stats": ([ctypes.POINTER(u64), ctypes.POINTER(u64), ctypes.POINTER(u64)], i32),
        "qs_jit_shutdown": ([], i32),
        "qs_begin_capture": ([vp], i32),
        "qs_end_capture": ([vp, ctypes.POINTER(vp)], i32),
        "qs_graph_launch": ([vp, vp], i32),
        "qs_graph_destroy": ([vp], i32),
    }
    for name, (args, res) in sig.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = res


def lib():
    """Load libqsb200.so (building it first if it is absent and nvcc exists)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            from . import build as _build

            _build.build()
        _lib = ctypes.CDLL(str(LIB_PATH))
        _declare(_lib)
        # stop the pass-compile threads before interpreter / library teardown
        import atexit

        atexit.register(_lib.qs_jit_shutdown)
    return _lib


def last_error() -> str:
    return lib().qs_last_error().decode(errors="replace")


def check(rc: int) -> None:
    if rc == QS_OK:
        return
    msg = last_error()
    if rc == QS_ERR_INDEX:
        raise IndexError(msg)
    if rc in (QS_ERR_VALUE, QS_ERR_NULL):
        raise ValueError(msg)
    if rc == QS_ERR_CAPACITY:
        raise CapacityError(msg)
    if rc == QS_ERR_DEGENERATE:
        raise DegenerateStateError(msg)
    raise DeviceError(msg)


def device_count() -> int:
    n = ctypes.c_int(0)
    rc = lib().qs_device_count(ctypes.byref(n))
    return n.value if rc == QS_OK else 0


def pcg_from_seed(seed) -> qs_pcg64:
    """numpy default_rng(seed)'s PCG64 state (the reference's draw source, measure.py:81).
    A Generator / BitGenerator seed is snapshotted, not advanced: the caller
    advances it with consume_draws() once the draws have been taken."""
    bg = np.random.default_rng(seed).bit_generator
    if not isinstance(bg, np.random.PCG64):
        raise TypeError(f"sampling draws from PCG64 (numpy's default_rng); got {type(bg).__name__}")
    st = bg.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return qs_pcg64((s >> 64) & m, s & m, (inc >> 64) & m, inc & m)


def consume_draws(seed, k: int) -> None:
    """pairsim draws rng.random(k) from default_rng(seed) (measure.py:81-82, 97):
    for a caller-owned Generator / BitGenerator that advances the caller's
    stream by k 64-bit outputs; ints and None leave nothing to advance."""
    if isinstance(seed, (np.random.Generator, np.random.BitGenerator)):
        np.random.default_rng(seed).bit_generator.advance(int(k))


def pinned_empty(count: int, dtype=np.float64) -> np.ndarray:
    """A numpy array in page-locked host memory (qs_host_alloc), freed when the
    array (and every view of it) is gone.  Readouts into it are plain DMA."""
    import weakref

    dt = np.dtype(dtype)
    nbytes = int(count) * dt.itemsize
    ptr = ctypes.c_void_p()
    check(lib().qs_host_alloc(nbytes, ctypes.byref(ptr)))
    buf = (ctypes.c_char * max(1, nbytes)).from_address(ptr.value)
    weakref.finalize(buf, lib().qs_host_free, ctypes.c_void_p(ptr.value))
    return np.frombuffer(buf, dtype=dt, count=int(count))


def f32ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def f64ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))
