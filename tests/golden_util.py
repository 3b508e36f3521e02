"""Helpers for replaying the pairsim golden fixtures (tests/golden/)."""

from __future__ import annotations

import hashlib
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden" / "pairsim_golden.npz"

_cache = None


def golden():
    global _cache
    if _cache is None:
        z = np.load(GOLDEN)
        _cache = {k: z[k] for k in z.files}
        _cache["meta"] = dict(zip(_cache["meta_keys"].tolist(), _cache["meta_vals"].tolist()))
    return _cache


def digest(arr: np.ndarray) -> str:
    if arr.dtype in (np.complex64, np.float32):
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


def same_values(x: np.ndarray, y: np.ndarray) -> bool:
    """Bit-exact up to the sign of zero (x == y elementwise, NaN-free)."""
    return x.shape == y.shape and bool(np.all(x == y))


def hist_from_outcomes(outcomes: np.ndarray):
    keys, counts = np.unique(outcomes, return_counts=True)
    return keys.astype(np.int64), counts.astype(np.int64)


_R = np.float32(1.0 / np.sqrt(2.0))
H_M8 = np.array([_R, 0, _R, 0, _R, 0, -_R, 0], np.float32)
X_M8 = np.array([0, 0, 1, 0, 1, 0, 0, 0], np.float32)
