"""CPU shard engine for the sharded-layer tests: the oracle (TEST INFRASTRUCTURE)
applied to a numpy complex64 shard.  Implements the engine interface of
paper_1805_00988_b200.sharded.CudaEngine."""

from __future__ import annotations

import numpy as np
import torch

from golden_util import M8Gate
from oracle import c as oc


class OracleEngine:
    def __init__(self, num_qubits: int):
        self.num_qubits = num_qubits
        self.amps = np.zeros(1 << num_qubits, np.complex64)

    def reset(self, basis):
        self.amps[:] = 0
        if basis is not None:
            self.amps[basis] = 1

    def apply(self, kind, target, ctrl_mask, m):
        g = M8Gate(m)
        ctrls = [q for q in range(64) if (ctrl_mask >> q) & 1]
        if not ctrls:
            oc.apply_gate(self.amps, target, g)
        elif len(ctrls) == 1:
            oc.apply_controlled_gate(self.amps, ctrls[0], target, g)
        elif len(ctrls) == 2:
            oc.apply_cc_gate(self.amps, ctrls[0], ctrls[1], target, g)
        else:
            raise NotImplementedError

    def apply_ops(self, ops, exact=True):
        for kind, t, cm, m in ops:
            self.apply(kind, t, cm, m)

    def swap_qubits(self, a, b):
        idx = np.arange(self.amps.size)
        ba, bb = (idx >> a) & 1, (idx >> b) & 1
        src = idx ^ ((ba ^ bb) << a) ^ ((ba ^ bb) << b)
        self.amps[:] = self.amps[src]

    def view(self):
        return torch.from_numpy(self.amps.view(np.float32))

    def comm_begin(self):
        pass

    def comm_end(self):
        pass

    def amplitudes(self):
        return self.amps.copy()

    def probabilities(self):
        return oc.probabilities(self.amps)

    def norm_squared(self):
        return float(oc.probabilities(self.amps).sum())

    def synchronize(self):
        pass

    def cdf_extend(self, start):
        return float(np.cumsum(np.concatenate([[start], oc.probabilities(self.amps)]))[-1])

    # peer-memory global gates: in one process the "peer reference" is the
    # partner engine itself; the same half split as csrc/peer.cu
    def peer_ref(self):
        return self

    def peer_gate(self, peer, own_is_a, ctrl_mask, m):
        L = self.num_qubits
        free = [q for q in range(L) if not (ctrl_mask >> q) & 1]
        idx = np.arange(1 << L)
        sel = (idx & ctrl_mask) == ctrl_mask
        if free:
            s = free[-1]
            sel &= ((idx >> s) & 1) == (0 if own_is_a else 1)
        elif not own_is_a:
            return
        i = idx[sel]
        va = (self.amps if own_is_a else peer.amps)[i]
        vb = (peer.amps if own_is_a else self.amps)[i]
        tmp = np.empty(2 * i.size, np.complex64)
        tmp[0::2], tmp[1::2] = va, vb
        oc.apply_gate(tmp, 0, M8Gate(m))
        (self.amps if own_is_a else peer.amps)[i] = tmp[0::2]
        (peer.amps if own_is_a else self.amps)[i] = tmp[1::2]

    def swap_peer(self, peer, own_off, peer_off, count):
        a = self.amps[own_off: own_off + count].copy()
        self.amps[own_off: own_off + count] = peer.amps[peer_off: peer_off + count]
        peer.amps[peer_off: peer_off + count] = a

    def sample_shard(self, k, rng, start, total, base, gdim, is_last):
        cdf = np.cumsum(np.concatenate([[start], oc.probabilities(self.amps)]))[1:]
        ncdf = cdf / total
        u = oc.pcg64_random_words((rng.state_hi, rng.state_lo, rng.inc_hi, rng.inc_lo), k)
        idx = np.searchsorted(ncdf, u, side="right")
        own = (u >= start / total) & (is_last | (ncdf[-1] > u))
        out = np.minimum(base + idx, gdim - 1)
        return np.where(own, out, -1).astype(np.int64)
