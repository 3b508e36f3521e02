"""Host model of the exact sampler's chunk-start resolution (csrc/measure.cu,
M3/M4): the sequential fp64 running sum of pairsim's cumsum
(pkg/src/pairsim/measure.py:69) reproduced from per-chunk trajectories and
composed parity maps.  Pure Python floats are IEEE doubles with
round-to-nearest-even, i.e. the device's __dadd_rn.

Checks the two facts the kernels rely on: (1) inside one binade a chunk
moves the bit pattern of the running value by inc[parity(s)], taken from its
trajectories from an even guess g0 and from g0 + ulp; (2) these maps compose
associatively, so a block reduces to one map and the chunk starts inside it
are block start + exclusive prefix map — equal to the sequential sums bit
for bit.
"""

from __future__ import annotations

import random
import struct

import pytest


def bits(x: float) -> int:
    return struct.unpack("<q", struct.pack("<d", x))[0]


def from_bits(b: int) -> float:
    return struct.unpack("<d", struct.pack("<q", b))[0]


def seq(s: float, ps) -> float:
    for p in ps:
        s = s + p
    return s


def compose(x, y):
    """x, then y (PMap of csrc/measure.cu)."""
    a0 = x[0] + (y[1] if x[0] & 1 else y[0])
    a1 = x[1] + (y[1] if (1 + x[1]) & 1 else y[0])
    return (a0, a1)


def chunk_map(g0: float, ps):
    """(inc0, inc1) from the two guessed trajectories (k_trajectories +
    k_block_maps); None when a trajectory leaves g0's binade."""
    g0 = from_bits(bits(g0) & ~1)
    g1 = from_bits(bits(g0) + 1)
    t0, t1 = seq(g0, ps), seq(g1, ps)
    e = bits(g0) >> 52
    if bits(t0) >> 52 != e or bits(t1) >> 52 != e:
        return None
    return (bits(t0) - bits(g0), bits(t1) - bits(g1))


def make_chunks(rng: random.Random, nch: int, csize: int, scale: float):
    return [[rng.random() * scale for _ in range(csize)] for _ in range(nch)]


@pytest.mark.parametrize("seed", range(6))
def test_chunk_maps_reproduce_sequential_sum(seed):
    rng = random.Random(seed)
    chunks = make_chunks(rng, 64, 16, 2.0 ** -40)
    s = 1.0 + rng.random() * 0.5  # inside [1, 2): one binade throughout
    for ch in chunks:
        guess = s + rng.choice([-1, 1]) * rng.random() * 2.0 ** -45  # a nearby guess, same binade
        m = chunk_map(guess, ch)
        assert m is not None
        want = seq(s, ch)
        got = from_bits(bits(s) + m[bits(s) & 1])
        assert bits(got) == bits(want)
        s = want


@pytest.mark.parametrize("seed", range(6))
def test_block_scan_equals_walk(seed):
    rng = random.Random(100 + seed)
    chunks = make_chunks(rng, 256, 8, 2.0 ** -38)
    s0 = 1.0 + rng.random() * 0.25
    # sequential walk: every chunk start
    starts, s = [], s0
    for ch in chunks:
        starts.append(s)
        s = seq(s, ch)
    end = s
    # per-chunk maps from guesses (here: the true starts perturbed), then an
    # inclusive scan in a random association order
    maps = []
    for st, ch in zip(starts, chunks):
        m = chunk_map(st + rng.random() * 2.0 ** -44, ch)
        assert m is not None
        maps.append(m)
    prefix = [(0, 0)]
    for m in maps:
        prefix.append(compose(prefix[-1], m))
    b0 = bits(s0)
    for k, st in enumerate(starts):
        assert bits(st) == b0 + prefix[k][b0 & 1]
    assert bits(end) == b0 + prefix[-1][b0 & 1]
    # associativity: a tree reduction gives the same block map
    def tree(ms):
        if len(ms) == 1:
            return ms[0]
        h = len(ms) // 2
        return compose(tree(ms[:h]), tree(ms[h:]))

    assert tree(maps) == prefix[-1]


def test_parity_matters():
    """Ties: an odd start can round differently from an even one, which is
    why each chunk carries two increments."""
    u = 2.0 ** -52
    ps = [u / 2] * 3  # every add is an exact tie at 1.0's grid
    even, odd = 1.0, 1.0 + u
    m = chunk_map(even, ps)
    assert bits(seq(even, ps)) - bits(even) == m[0]
    assert bits(seq(odd, ps)) - bits(odd) == m[1]
    assert m[0] != m[1]
