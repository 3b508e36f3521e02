"""The sharded exchange alone vs a D2D copy (bench extras' exchange_alone leg)."""
import json, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent.parent))
import torch
from paper_1805_00988_b200.sharded import ShardedState
from paper_1805_00988_b200 import _native as _N
payload = 2 * (1 << 29) * 8
out = {}
for mode, exch in (("copy_exchange", "nccl"), ("peer_swap_kernel", "peer")):
    vs = ShardedState.virtual(31, 2, peer_gates=False, exchange=exch)
    vs._exchange(0); vs.synchronize()
    t0 = time.perf_counter()
    for _ in range(4):
        vs._exchange(0)
    vs.synchronize()
    dt = (time.perf_counter() - t0) / 4
    out[mode] = {"ms": dt * 1e3, "payload_GBps": payload / dt / 1e9}
    vs.close(); _N.lib().qs_release_cached(-1)
a = torch.empty(payload // 4, device="cuda"); b = torch.empty_like(a); b.copy_(a); torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(4):
    b.copy_(a)
torch.cuda.synchronize()
out["d2d"] = (time.perf_counter() - t0) / 4 * 1e3
print(json.dumps(out))
