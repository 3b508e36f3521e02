"""TEST INFRASTRUCTURE: numpy port of the reference's CPU hot path.

A restatement of pairsim's vectorised pair sweep and measure path, with the
same numpy operations in the same order so it runs at the reference's speed
and (on an FMA host) produces the reference's bits:

* nth_cleared            pkg/src/pairsim/kernel.py:31-37
* ThreadExecutor chunks  pkg/src/pairsim/kernel.py:56-89 (contiguous chunks of
                         ceil(items/workers); inline below 2^16 items)
* apply_gate             pkg/src/pairsim/kernel.py:108-132
* apply_controlled_gate  pkg/src/pairsim/kernel.py:135-165
* probabilities          pkg/src/pairsim/measure.py:29-34
* sample                 pkg/src/pairsim/measure.py:68-85

bench.py times this port as the CPU baseline (``cpu_baseline.kind = "port"``)
because /root/reference does not exist on the GPU box.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np


def nth_cleared(i, target):
    mask = (1 << target) - 1
    return (i & mask) | ((i & ~mask) << 1)


class Executor:
    """kernel.py:56-89 — contiguous chunks on a thread pool, full barrier."""

    def __init__(self, workers: int | None = None, min_parallel_items: int = 1 << 16):
        self.workers = workers or min(os.cpu_count() or 1, 8)
        self.min_parallel_items = min_parallel_items
        self._pool = None

    def run(self, n_items: int, body) -> None:
        if self.workers == 1 or n_items < self.min_parallel_items:
            body(0, n_items)
            return
        if self._pool is None:
            self._pool = ThreadPoolExecutor(max_workers=self.workers)
        chunk = -(-n_items // self.workers)
        futures = [self._pool.submit(body, lo, min(lo + chunk, n_items)) for lo in range(0, n_items, chunk)]
        for f in futures:
            f.result()

    def close(self) -> None:
        if self._pool is not None:
            self._pool.shutdown(wait=True)
            self._pool = None


def _entries(amps: np.ndarray, gate):
    scalar = amps.dtype.type
    return tuple(scalar(x) for x in (gate.a, gate.b, gate.c, gate.d))


def apply_gate(amps: np.ndarray, target: int, gate, executor: Executor) -> np.ndarray:
    n = int(amps.size).bit_length() - 1
    ga, gb, gc, gd = _entries(amps, gate)
    tbit = 1 << target

    def body(lo, hi):
        i = np.arange(lo, hi, dtype=np.int64)
        a = nth_cleared(i, target)
        b = a | tbit
        va = amps[a]
        vb = amps[b]
        amps[a] = ga * va + gb * vb
        amps[b] = gd * vb + gc * va

    executor.run(1 << (n - 1), body)
    return amps


def apply_controlled_gate(amps: np.ndarray, control: int, target: int, gate, executor: Executor) -> np.ndarray:
    n = int(amps.size).bit_length() - 1
    ga, gb, gc, gd = _entries(amps, gate)
    tbit, cbit = 1 << target, 1 << control

    def body(lo, hi):
        i = np.arange(lo, hi, dtype=np.int64)
        a = nth_cleared(i, target)
        a = a[(a & cbit) != 0]
        b = a | tbit
        va = amps[a]
        vb = amps[b]
        amps[a] = ga * va + gb * vb
        amps[b] = gd * vb + gc * va

    executor.run(1 << (n - 1), body)
    return amps


def probabilities(amps: np.ndarray) -> np.ndarray:
    re = amps.real.astype(np.float64, copy=False)
    im = amps.imag.astype(np.float64, copy=False)
    return re * re + im * im


def sample_outcomes(amps: np.ndarray, k: int, seed) -> np.ndarray:
    cdf = np.cumsum(probabilities(amps))
    total = cdf[-1]
    if total <= 0.0:
        raise ZeroDivisionError("degenerate state")
    cdf = cdf / total
    draws = np.random.default_rng(seed).random(k)
    out = np.searchsorted(cdf, draws, side="right")
    np.minimum(out, amps.size - 1, out=out)
    return out
