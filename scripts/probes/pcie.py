"""Host<->device copy rates of this box for the e2e leg: pinned H2D alone, D2H
alone, both at once on two streams, and the e2e pipeline variants through the
C ABI (qs_set/get_amplitudes_async) with R registers in flight."""

import json
import sys
import time

import torch

from paper_1805_00988_b200 import State, build_hadamard_layer, fusion
from paper_1805_00988_b200.circuits import lower_ops

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
nb = 8 << n
dev = torch.device("cuda:0")
h_in = torch.empty(nb // 4, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(nb // 4, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(nb // 4, dtype=torch.float32, device=dev)
d_b = torch.empty(nb // 4, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
res = {}


def t(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t0)
    return best


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn in [("h2d", h2d), ("d2h", d2h), ("both", both)]:
    dt = t(fn)
    res[name] = {"s": dt, "GB/s per direction": nb / dt / 1e9}
del d_a, d_b
torch.cuda.empty_cache()

passes = fusion.plan(n, lower_ops(build_hadamard_layer(n)))


def pipeline(R, K):
    regs = [State(n) for _ in range(R)]
    strs = [torch.cuda.ExternalStream(r.stream()) for r in regs]
    outs = [torch.empty(nb // 4, dtype=torch.float32, pin_memory=True) for _ in range(min(R, 2))]
    up_ev = [torch.cuda.Event() for _ in range(K + 8)]
    dn_ev = [torch.cuda.Event() for _ in range(K + 8)]

    def run(K):
        for k in range(K):
            i = k % R
            s, st = regs[i], strs[i]
            if k:
                st.wait_event(up_ev[k - 1])
            s.upload_async(h_in.data_ptr())
            up_ev[k].record(st)
            fusion.run(s, passes)
            if k:
                st.wait_event(dn_ev[k - 1])
            s.download_async(outs[k % len(outs)].data_ptr())
            dn_ev[k].record(st)
        for s in regs:
            s.flush()

    run(2)
    fusion.jit_sync()
    run(2)
    t0 = time.perf_counter()
    run(K)
    dt = time.perf_counter() - t0
    for r in regs:
        r.close()
    return {"ms_per_step": dt / K * 1e3, "gates/s": K * n / dt}


for R in (2, 3):
    for K in (3, 6, 10):
        res[f"pipe_R{R}_K{K}"] = pipeline(R, K)
print(json.dumps(res, indent=1))
