"""TEST INFRASTRUCTURE: ctypes binding of oracle/qsim_oracle.c (liboracle.so).

Each function cites the reference function it restates; arrays are complex64
(or complex128: the *_d restatements) numpy arrays mutated in place, exactly
like pairsim's StateVector.amps.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

_lib = None


def build() -> Path:
    src = HERE / "qsim_oracle.c"
    if not LIB_PATH.exists() or LIB_PATH.stat().st_mtime < src.stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(str(LIB_PATH))
        f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
        f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
        i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
        u64 = ctypes.c_uint64
        L.oracle_nth_cleared.argtypes = [u64, ctypes.c_int]
        L.oracle_nth_cleared.restype = u64
        L.oracle_apply_gate.argtypes = [f32p, ctypes.c_int, ctypes.c_int, f32p]
        L.oracle_apply_controlled_gate.argtypes = [f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, f32p]
        L.oracle_apply_cc_gate.argtypes = [f32p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, f32p]
        L.oracle_probabilities.argtypes = [f32p, ctypes.c_int, f64p]
        L.oracle_pcg64_random.argtypes = [u64, u64, u64, u64, ctypes.c_int64, f64p]
        L.oracle_sample.argtypes = [f32p, ctypes.c_int, u64, u64, u64, u64, ctypes.c_int64, i64p]
        L.oracle_sample.restype = ctypes.c_int
        L.oracle_apply_gate_d.argtypes = [f64p, ctypes.c_int, u64, ctypes.c_int, f64p]
        L.oracle_probabilities_d.argtypes = [f64p, ctypes.c_int, f64p]
        L.oracle_sample_d.argtypes = [f64p, ctypes.c_int, u64, u64, u64, u64, ctypes.c_int64, i64p]
        L.oracle_sample_d.restype = ctypes.c_int
        _lib = L
    return _lib


def gate_m8(gate) -> np.ndarray:
    """[[a,b],[c,d]] -> float32[8], rounded like np.complex64(x) (kernel.py:118-119)."""
    vals = [np.complex64(complex(x)) for x in (gate.a, gate.b, gate.c, gate.d)]
    return np.array([v for c in vals for v in (c.real, c.imag)], dtype=np.float32)


def gate_m8d(gate) -> np.ndarray:
    """[[a,b],[c,d]] -> float64[8] (np.complex128(x) of a Python complex is exact)."""
    vals = [complex(x) for x in (gate.a, gate.b, gate.c, gate.d)]
    return np.array([v for c in vals for v in (c.real, c.imag)], dtype=np.float64)


def _is_double(amps: np.ndarray) -> bool:
    return amps.dtype == np.complex128


def _f64view(amps: np.ndarray) -> np.ndarray:
    assert amps.dtype == np.complex128 and amps.flags.c_contiguous
    return amps.view(np.float64)


def _f32view(amps: np.ndarray) -> np.ndarray:
    assert amps.dtype == np.complex64 and amps.flags.c_contiguous
    return amps.view(np.float32)


def nth_cleared(i: int, target: int) -> int:
    return int(lib().oracle_nth_cleared(i, target))


def apply_gate(amps: np.ndarray, target: int, gate) -> np.ndarray:
    n = int(amps.size).bit_length() - 1
    if _is_double(amps):
        lib().oracle_apply_gate_d(_f64view(amps), n, 0, target, gate_m8d(gate))
    else:
        lib().oracle_apply_gate(_f32view(amps), n, target, gate_m8(gate))
    return amps


def apply_controlled_gate(amps: np.ndarray, control: int, target: int, gate) -> np.ndarray:
    n = int(amps.size).bit_length() - 1
    if _is_double(amps):
        lib().oracle_apply_gate_d(_f64view(amps), n, 1 << control, target, gate_m8d(gate))
    else:
        lib().oracle_apply_controlled_gate(_f32view(amps), n, control, target, gate_m8(gate))
    return amps


def apply_cc_gate(amps: np.ndarray, c1: int, c2: int, target: int, gate) -> np.ndarray:
    n = int(amps.size).bit_length() - 1
    if _is_double(amps):
        lib().oracle_apply_gate_d(_f64view(amps), n, (1 << c1) | (1 << c2), target, gate_m8d(gate))
    else:
        lib().oracle_apply_cc_gate(_f32view(amps), n, c1, c2, target, gate_m8(gate))
    return amps


def probabilities(amps: np.ndarray) -> np.ndarray:
    n = int(amps.size).bit_length() - 1
    out = np.empty(amps.size, dtype=np.float64)
    if _is_double(amps):
        lib().oracle_probabilities_d(_f64view(amps), n, out)
    else:
        lib().oracle_probabilities(_f32view(amps), n, out)
    return out


def pcg_words(seed):
    """numpy default_rng(seed) PCG64 state as (state_hi, state_lo, inc_hi, inc_lo)."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return (s >> 64) & m, s & m, (inc >> 64) & m, inc & m


def pcg64_random(seed, k: int) -> np.ndarray:
    return pcg64_random_words(pcg_words(seed), k)


def pcg64_random_words(words, k: int) -> np.ndarray:
    out = np.empty(k, dtype=np.float64)
    lib().oracle_pcg64_random(*[int(w) for w in words], k, out)
    return out


def sample_outcomes(amps: np.ndarray, k: int, seed) -> np.ndarray:
    """Per-draw outcomes of pairsim.measure.sample (measure.py:76-85)."""
    n = int(amps.size).bit_length() - 1
    out = np.empty(k, dtype=np.int64)
    if _is_double(amps):
        rc = lib().oracle_sample_d(_f64view(amps), n, *pcg_words(seed), k, out)
    else:
        rc = lib().oracle_sample(_f32view(amps), n, *pcg_words(seed), k, out)
    if rc == 4:
        raise ZeroDivisionError("degenerate state")
    if rc != 0:
        raise MemoryError("oracle_sample allocation failed")
    return out
