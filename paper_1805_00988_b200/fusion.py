"""Pass planner: groups a gate sequence into fused HBM passes (qs_apply_fused).

Each pass names a tile qubit set Q (|Q| = K, always containing qubits 0..5
so every tile is made of 512-byte contiguous segments) and takes ops in
circuit order while:

* a PAIR op's target is in Q, or Q still has room to add it, and
* a PHASE op (diagonal, a == 1, b == c == 0: u1/z/s/t and their controlled
  forms) is always absorbable — it is an element-wise multiply with its
  target/control bits as a predicate, wherever those bits live.

Ops are never reordered, so the fused result is the same as the sequential
one (kernel.py:244-245 barrier semantics preserved by construction).  A pass
holding a single op is dispatched to the plain sweep kernels instead (the
phase kernel touches fewer bytes than a full tile pass).
"""

from __future__ import annotations

import weakref
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .gates import cached_ptr, entries_ptr, is_phase

LOW = 6


@dataclass
class Pass:
    tile: list[int]
    ops: list[tuple[int, int, int, np.ndarray]] = field(default_factory=list)  # (kind, target, ctrl_mask, m8)

    def op_array(self) -> np.ndarray:
        """qs_op records (float32 entries) or qs_op64 (float64, complex128 registers)."""
        double = bool(self.ops) and self.ops[0][3].dtype == np.float64
        arr = np.zeros(len(self.ops), dtype=N.OP64_DTYPE if double else N.OP_DTYPE)
        for i, (kind, t, cm, m) in enumerate(self.ops):
            arr[i]["kind"] = kind
            arr[i]["target"] = t
            arr[i]["ctrl_mask"] = cm
            arr[i]["m"] = m
        return arr


_KIND: dict = {}  # id(cached entries array) -> QS_OP_PHASE / QS_OP_PAIR


def lower(gate, target: int, controls=(), double: bool = False) -> tuple[int, int, int, np.ndarray]:
    m = entries_ptr(gate, double)[0]  # read-only, shared by every op of the same gate
    cm = 0
    for c in controls:
        cm |= 1 << int(c)
    kind = _KIND.get(id(m))
    if kind is None:
        kind = N.QS_OP_PHASE if is_phase(m) else N.QS_OP_PAIR
        if cached_ptr(m) is not None:  # cached array: remember its kind while it lives
            _KIND[id(m)] = kind
            weakref.finalize(m, _KIND.pop, id(m), None)
    return kind, int(target), cm, m


def default_tile_qubits(num_qubits: int) -> int:
    return min(13, num_qubits)


def plan(num_qubits: int, ops, tile_qubits: int | None = None, reorder: bool = False) -> list[Pass]:
    """Greedy in-order grouping into passes of at most K tile qubits.  Without
    an explicit K: 12-qubit tiles (two persistent CTAs per SM) unless those
    need more than 25% more passes than 13-qubit ones.  (Measured on B200
    with the dynamic tile scheduler, scripts/qft_passes.py: QFT(28) 8.5 ms
    on 12-qubit tiles vs 9.3 ms on 13, QFT(30) 36.3 vs 37.5 ms.)

    reorder=True (opt-in, QSB_FUSE_REORDER=1 for execute()): the
    commutation-aware planner _plan_reorder — gates on disjoint qubits are
    exchanged freely.  That is exact in real arithmetic but NOT bit-exact in
    floating point (e.g. H(a) H(b) sums (v0 + v1) + (v2 + v3) where H(b) H(a)
    sums (v0 + v2) + (v1 + v3)), so results agree with the reference to
    rounding (tested at rtol 1e-5, the north_star bar) instead of bit for
    bit.  The default planner only moves permutations, which is exact.  With
    reorder=True the in-order plan is still used when it needs no more
    passes (QFT: the reordered plan pulls later rows' phases forward into
    heavier passes for no pass saved)."""
    def choose(pl):
        if tile_qubits is None and num_qubits >= 13:
            p13 = pl(num_qubits, ops, 13)
            p12 = pl(num_qubits, ops, 12)
            return p12 if 4 * len(p12) <= 5 * len(p13) else p13
        return pl(num_qubits, ops, tile_qubits)

    ops = list(ops)
    base = choose(_plan)
    if not reorder:
        return base
    alt = choose(_plan_reorder)
    return alt if len(alt) < len(base) else base


def _plan_reorder(num_qubits: int, ops, tile_qubits: int | None) -> list[Pass]:
    """Commutation-aware grouping: ops form a DAG (an op depends on the
    latest earlier op sharing any qubit with it); a pass absorbs every READY
    op that fits its tile (diagonal ops always, pair ops whose target is a
    tile qubit), and while the tile has room it adds the qubit whose
    addition unlocks the most ops (simulated absorption over the DAG).  Ops
    sharing a qubit keep their order, so each qubit's gate sequence is the
    circuit's."""
    n = num_qubits
    K = tile_qubits or default_tile_qubits(n)
    if n < 10 or K < 10:
        return [Pass(list(range(n)), list(ops))] if ops else []
    ops = list(ops)
    m = len(ops)
    masks = [_qubits(op) for op in ops]
    # successors through each op's qubits: op j waits for the latest earlier op on each of its qubits
    last = {}
    preds = [0] * m
    succ = [[] for _ in range(m)]
    for j, mk in enumerate(masks):
        ps = set()
        q = mk
        while q:
            b = q & -q
            i = last.get(b)
            if i is not None:
                ps.add(i)
            last[b] = j
            q ^= b
        preds[j] = len(ps)
        for i in ps:
            succ[i].append(j)
    done = [False] * m
    ready = {j for j in range(m) if preds[j] == 0}

    def fits(j, tile):
        kind, t = ops[j][0], ops[j][1]
        return kind != N.QS_OP_PAIR or (tile >> t) & 1

    def absorb(tile, rd, pc, dn, out):
        """Take every ready op that fits, transitively (simulation when out is None)."""
        stack = [j for j in rd if fits(j, tile)]
        count = 0
        while stack:
            j = stack.pop()
            if dn[j] or j not in rd:
                continue
            rd.discard(j)
            dn[j] = True
            count += 1
            if out is not None:
                out.append(j)
            for k in succ[j]:
                pc[k] -= 1
                if pc[k] == 0:
                    rd.add(k)
                    if fits(k, tile):
                        stack.append(k)
        return count

    base = (1 << min(LOW, n)) - 1
    passes: list[Pass] = []
    remaining = m
    while remaining:
        tile = base
        taken: list[int] = []
        remaining -= absorb(tile, ready, preds, done, taken)
        while remaining and bin(tile).count("1") < K:
            cands = {ops[j][1] for j in ready if ops[j][0] == N.QS_OP_PAIR and not (tile >> ops[j][1]) & 1}
            if not cands:
                break
            best, best_gain = None, -1
            for q in sorted(cands):
                gain = absorb(tile | (1 << q), set(ready), list(preds), list(done), None)
                if gain > best_gain:
                    best, best_gain = q, gain
            tile |= 1 << best
            remaining -= absorb(tile, ready, preds, done, taken)
        taken.sort()  # circuit order among independent ops (the DAG order holds: sorted is a topological order)
        qs = [q for q in range(n) if (tile >> q) & 1]
        extra = [q for q in range(n - 1, -1, -1) if not (tile >> q) & 1]
        qs.extend(extra[: max(0, K - len(qs))])
        qs.sort()
        passes.append(Pass(qs, _order_for_stages([ops[j] for j in taken], qs)))
    return passes


def _order_for_stages(pops, tile) -> list:
    """Reorder a reordered pass's ops (DAG order kept: ops sharing a qubit
    stay in order) so that the kernel's stage planner (csrc/fused.cu
    plan_pass: a stage holds its pair targets in RB register bits and
    leaves one f-bit of each class {0,5} / {1,6} / {2,7} to the lanes) needs as
    few stages as possible: every stage is a shared-memory round trip of
    the whole tile (~3 ms per extra stage at 32 qubits).  Greedy: absorb
    every ready op whose target bit is in the current register set; grow the
    set by the bit that unlocks the most ops; else start a new stage."""
    m = len(pops)
    if m < 3:
        return pops
    local = {q: i for i, q in enumerate(tile)}
    nphase = sum(1 for op in pops if op[0] != N.QS_OP_PAIR)
    RB = 3 if 2 * nphase > m else 4

    def fbit(op):
        kind, t = op[0], op[1]
        if kind != N.QS_OP_PAIR:
            return None
        lb = local.get(t)
        return None if lb is None or lb == 0 else lb - 1

    nf = len(tile) - 1

    def triple_ok(rs):  # one free f-bit in each class {0,5}, {1,6}, {2,7} (csrc/fused.cu)
        return all(c not in rs or (c + 5 < nf and c + 5 not in rs) for c in range(3))

    masks = [_qubits(op) for op in pops]
    preds = [0] * m
    succ = [[] for _ in range(m)]
    last = {}
    for j, mk in enumerate(masks):
        ps = set()
        q = mk
        while q:
            b = q & -q
            if b in last:
                ps.add(last[b])
            last[b] = j
            q ^= b
        preds[j] = len(ps)
        for i in ps:
            succ[i].append(j)
    fb = [fbit(op) for op in pops]
    ready = {j for j in range(m) if preds[j] == 0}
    out: list = []

    def absorb(regs, rd, pc, sim):
        stack = [j for j in rd if fb[j] is None or fb[j] in regs]
        got = 0
        while stack:
            j = stack.pop()
            if j not in rd:
                continue
            rd.discard(j)
            got += 1
            if not sim:
                out.append(j)
            for k in succ[j]:
                pc[k] -= 1
                if pc[k] == 0:
                    rd.add(k)
                    if fb[k] is None or fb[k] in regs:
                        stack.append(k)
        return got

    regs: set = set()
    while len(out) < m:
        absorb(regs, ready, preds, False)
        if len(out) == m:
            break
        cands = {fb[j] for j in ready if fb[j] is not None and fb[j] not in regs}
        cands = [f for f in cands if len(regs) < RB and triple_ok(regs | {f})]
        if not cands:
            regs = set()  # next stage
            continue
        best = max(sorted(cands), key=lambda f: absorb(regs | {f}, set(ready), list(preds), True))
        regs = regs | {best}
    # keep circuit order inside each maximal run the greedy emitted (cosmetic)
    return [pops[j] for j in out]


def is_permutation(m: np.ndarray) -> bool:
    """X (b == c == 1, a == d == 0 exactly): with any controls, a basis
    permutation — it moves amplitudes without arithmetic."""
    return bool(m[0] == 0 and m[1] == 0 and m[2] == 1 and m[3] == 0 and m[4] == 1 and m[5] == 0
                and m[6] == 0 and m[7] == 0)


def _qubits(op) -> int:
    kind, t, cm, _ = op
    return cm | (1 << t)


def _plan(num_qubits: int, ops, tile_qubits: int | None, defer: bool = True) -> list[Pass]:
    """Greedy grouping in circuit order.  One exact reordering is allowed: a
    permutation op (X / CX / CCX) whose target does not fit the current tile
    is deferred past later ops that touch none of its qubits — a permutation
    only relocates amplitudes, so it commutes bit for bit with any gate on
    disjoint qubits — and lands in the next pass.  Every other op keeps its
    place relative to every op it shares a qubit with."""
    n = num_qubits
    K = tile_qubits or default_tile_qubits(n)
    if n < 10 or K < 10:
        return [Pass(list(range(n)), list(ops))] if ops else []
    from collections import deque

    base = list(range(min(LOW, n)))
    passes: list[Pass] = []
    cur = Pass(list(base))
    queue = deque(ops)
    deferred: list = []
    dmask = 0  # qubits touched by the deferred ops

    def close():
        nonlocal cur, deferred, dmask
        if cur.ops:
            passes.append(cur)
        cur = Pass(list(base))
        queue.extendleft(reversed(deferred))
        deferred, dmask = [], 0

    while queue or deferred:
        if not queue:  # only deferred ops left: they start the next pass
            close()
            continue
        op = queue.popleft()
        kind, t = op[0], op[1]
        fits = kind != N.QS_OP_PAIR or t in cur.tile or len(cur.tile) < K
        if fits and not (_qubits(op) & dmask):
            if kind == N.QS_OP_PAIR and t not in cur.tile:
                cur.tile.append(t)
            cur.ops.append(op)
        elif defer and kind == N.QS_OP_PAIR and is_permutation(op[3]) and len(deferred) < 64 and cur.ops:
            deferred.append(op)
            dmask |= _qubits(op)
        else:
            queue.appendleft(op)
            close()
    if cur.ops:
        passes.append(cur)
    for p in passes:  # pad the tile to K qubits (extra qubits are free)
        extra = [q for q in range(n - 1, -1, -1) if q not in p.tile]
        p.tile.extend(extra[: max(0, K - len(p.tile))])
        p.tile.sort()
    return passes


def jit_sync(device: int = -1) -> None:
    """Wait until every queued pass program has compiled and is loaded (the
    passes run on the interpreter kernel until then, with the same bits)."""
    N.check(N.lib().qs_jit_sync(int(device)))


def jit_stats() -> dict:
    """{"compiled", "cache_hits", "failed"}: pass programs built with NVRTC by
    this process, loaded from the on-disk program cache, failed."""
    import ctypes

    c, h, f = ctypes.c_uint64(), ctypes.c_uint64(), ctypes.c_uint64()
    N.check(N.lib().qs_jit_stats(ctypes.byref(c), ctypes.byref(h), ctypes.byref(f)))
    return {"compiled": c.value, "cache_hits": h.value, "failed": f.value}


def run(state, passes: list[Pass], combine: bool = False, from_basis: int | None = None,
        chunk_sums: bool = False) -> bool:
    """Launch the planned passes on a State (asynchronous on its stream).
    combine=True: runs of unit-modulus diagonal ops as one product per
    amplitude (State.apply_fused; not bit-exact).  from_basis=b: the register
    starts as |b> (State.reset(b)), folded into the first pass when it is a
    fused one — its tiles are written as |b> instead of loaded.
    chunk_sums=True (after State.sample_prepare): the last pass, when it is a
    fused one, also leaves the sampler's chunk sums; returns whether it did."""
    last = len(passes) - 1
    sums = False
    for i, p in enumerate(passes):
        want = chunk_sums and i == last and len(p.ops) > 1
        extra = {"chunk_sums": True} if want else {}  # (shard objects take the plain signature)
        if i == 0 and from_basis is not None:
            if len(p.ops) > 1:
                state.apply_fused(p.tile, p.op_array(), combine=combine, from_basis=from_basis, **extra)
                sums = want
                continue
            state.reset(int(from_basis))
        if len(p.ops) == 1:
            kind, t, cm, m = p.ops[0]
            _single(state, kind, t, cm, m)
        else:
            state.apply_fused(p.tile, p.op_array(), combine=combine, **extra)
            sums = want
    if not passes and from_basis is not None:
        state.reset(int(from_basis))
    return sums


def _single(state, kind, t, cm, m) -> None:
    """One op: the dedicated sweep kernels (the phase kernel for diagonal ops)."""
    L = N.lib()
    ctrls = []
    while cm and len(ctrls) < 3:
        low = cm & -cm
        ctrls.append(low.bit_length() - 1)
        cm ^= low
    cm |= sum(1 << q for q in ctrls)
    mp = cached_ptr(m)  # entries arrays from lower() carry a cached pointer
    if m.dtype == np.float64:  # fp64 entries (complex128 registers)
        if mp is None:
            mp = N.f64ptr(np.ascontiguousarray(m))
        g1, g2, g3 = L.qs_apply_gate_f64, L.qs_apply_controlled_gate_f64, L.qs_apply_controlled_controlled_gate_f64
    else:
        if mp is None:
            mp = N.f32ptr(np.ascontiguousarray(m, dtype=np.float32))
        g1, g2, g3 = L.qs_apply_gate, L.qs_apply_controlled_gate, L.qs_apply_controlled_controlled_gate
    if not ctrls:
        N.check(g1(state.handle, t, mp))
    elif len(ctrls) == 1:
        N.check(g2(state.handle, ctrls[0], t, mp))
    elif len(ctrls) == 2:
        N.check(g3(state.handle, ctrls[0], ctrls[1], t, mp))
    else:  # >2 controls: a one-op pass (the library dispatches it to the sweep kernel)
        op = np.zeros(1, dtype=N.OP64_DTYPE if m.dtype == np.float64 else N.OP_DTYPE)
        op[0]["kind"], op[0]["target"], op[0]["ctrl_mask"], op[0]["m"] = kind, t, cm, m
        state.apply_fused([t], op)
