"""The paper's benchmark methodology (Algorithm 2; pairsim
bench.py:98-123) with the B200 backend registered beside the CPU reference.

For each width 1..max_qubits every back-end gets one untimed warm-up, then
`samples` trials pick a back-end uniformly at random (seeded) and time one
QFT(width) run end to end (register allocation + every gate + device barrier,
as the paper's bench_qcgpu times through queue.finish()).
Writes `simulator,qubits,seconds` CSV rows and a Welch t-test per width.

    python scripts/paper_algorithm2.py --max-qubits 24 --samples 10 --out profiles/alg2.csv
"""

from __future__ import annotations

import argparse
import csv
import math
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))


def b200_qft_runner(fuse: bool):
    from paper_1805_00988_b200 import State, build_qft, execute

    cache = {}

    def run(n: int) -> None:
        circ = cache.get(n) or cache.setdefault(n, build_qft(n))
        s = State(n)
        execute(circ, s, fuse=fuse)
        s.flush()
        s.close()

    return run


def cpu_qft_runner(workers):
    """pairsim's engine_qft_runner (bench.py:52-69) on the numpy port."""
    from oracle import port
    from paper_1805_00988_b200 import build_qft
    from paper_1805_00988_b200.circuits import Apply

    ex = port.Executor(workers=workers)

    def run(n: int) -> None:
        amps = np.zeros(1 << n, np.complex64)
        amps[0] = 1
        for ins in build_qft(n).instructions:
            if isinstance(ins, Apply):
                port.apply_gate(amps, ins.target, ins.gate, ex)
            else:
                port.apply_controlled_gate(amps, ins.control, ins.target, ins.gate, ex)

    return run


def welch(xs, ys):
    from scipy import stats

    if len(xs) < 2 or len(ys) < 2:
        return math.nan, math.nan
    r = stats.ttest_ind(xs, ys, equal_var=False)
    return float(r.statistic), float(r.pvalue)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--max-qubits", type=int, default=22)
    ap.add_argument("--samples", type=int, default=10)
    ap.add_argument("--seed", type=int, default=2018)
    ap.add_argument("--cpu-max-qubits", type=int, default=22)
    ap.add_argument("--out", default="gpurun_out/alg2.csv")
    args = ap.parse_args()
    import os

    backends = {"b200-fused": b200_qft_runner(True), "b200-unfused": b200_qft_runner(False),
                "cpu-port": cpu_qft_runner(len(os.sched_getaffinity(0)))}
    rng = np.random.default_rng(args.seed)
    labels = sorted(backends)
    records = []
    for width in range(1, args.max_qubits + 1):
        active = [l for l in labels if not (l == "cpu-port" and width > args.cpu_max_qubits)]
        for label in active:
            backends[label](width)  # warm-up (queues the B200 pass programs' compiles)
        from paper_1805_00988_b200 import fusion

        fusion.jit_sync()
        for _ in range(args.samples * len(active)):  # ~samples trials per back-end
            label = active[int(rng.integers(len(active)))]
            t0 = time.perf_counter()
            backends[label](width)
            records.append((label, width, time.perf_counter() - t0))
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    with open(args.out, "w", newline="") as fh:
        w = csv.writer(fh)
        w.writerow(["simulator", "qubits", "seconds"])
        w.writerows(records)
    print("width  b200-fused(ms)  b200-unfused(ms)  cpu-port(ms)  speedup  welch_p(fused vs cpu)")
    for width in range(1, args.max_qubits + 1):
        t = {l: [s for (lab, n, s) in records if lab == l and n == width] for l in labels}
        mean = {l: (1e3 * sum(v) / len(v) if v else math.nan) for l, v in t.items()}
        _, p = welch(t["b200-fused"], t["cpu-port"])
        sp = mean["cpu-port"] / mean["b200-fused"] if t["cpu-port"] and t["b200-fused"] else math.nan
        print(f"{width:5d}  {mean['b200-fused']:14.3f}  {mean['b200-unfused']:16.3f}  {mean['cpu-port']:12.3f}"
              f"  {sp:7.1f}  {p:.3g}")


if __name__ == "__main__":
    main()
