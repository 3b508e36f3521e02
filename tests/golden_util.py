"""Helpers for replaying the pairsim golden fixtures (tests/golden/)."""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden" / "pairsim_golden.npz"
GOLDEN_DOUBLE = Path(__file__).resolve().parent / "golden" / "pairsim_golden_double.npz"

_cache = {}


def _load(path):
    if path not in _cache:
        z = np.load(path)
        d = {k: z[k] for k in z.files}
        d["meta"] = dict(zip(d["meta_keys"].tolist(), d["meta_vals"].tolist()))
        _cache[path] = d
    return _cache[path]


def golden():
    """complex64 (Precision.SINGLE) fixtures: tests/golden/make_golden.py"""
    return _load(GOLDEN)


def golden_double():
    """complex128 (Precision.DOUBLE) fixtures: tests/golden/make_golden_double.py"""
    return _load(GOLDEN_DOUBLE)


def digest(arr: np.ndarray) -> str:
    if arr.dtype in (np.complex64, np.float32, np.complex128, np.float64):
        arr = arr + arr.dtype.type(0)
    return hashlib.sha256(np.ascontiguousarray(arr).tobytes()).hexdigest()


class M8Gate:
    """Minimal gate view over a float32[8] matrix (already complex64-rounded)."""

    def __init__(self, m8):
        m8 = np.asarray(m8, np.float32)
        self.m8 = m8
        self.a = complex(m8[0], m8[1])
        self.b = complex(m8[2], m8[3])
        self.c = complex(m8[4], m8[5])
        self.d = complex(m8[6], m8[7])


class M8DGate:
    """Gate view over fp64 (a, b, c, d) entries (complex128 registers)."""

    def __init__(self, m8):
        m8 = np.asarray(m8, np.float64)
        self.m8 = m8
        self.a = complex(m8[0], m8[1])
        self.b = complex(m8[2], m8[3])
        self.c = complex(m8[4], m8[5])
        self.d = complex(m8[6], m8[7])


def same_values(x: np.ndarray, y: np.ndarray) -> bool:
    """Bit-exact up to the sign of zero (x == y elementwise, NaN-free)."""
    return x.shape == y.shape and bool(np.all(x == y))


def hist_from_outcomes(outcomes: np.ndarray):
    keys, counts = np.unique(outcomes, return_counts=True)
    return keys.astype(np.int64), counts.astype(np.int64)


_R = np.float32(1.0 / np.sqrt(2.0))
H_M8 = np.array([_R, 0, _R, 0, _R, 0, -_R, 0], np.float32)
X_M8 = np.array([0, 0, 1, 0, 1, 0, 0, 0], np.float32)
