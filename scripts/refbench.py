"""The reference's own CPU path, timed beside the B200 backend (bench.py).

pairsim (the reference package) is pip-installed, unmodified, into
baseline/_ref (git-ignored; it travels to the GPU box with the snapshot):

    python -m pip install --no-index --no-build-isolation --no-deps \
        --target baseline/_ref <copy of /root/reference/pkg>

Nothing here reads /root/reference.  When baseline/_ref is missing the
callers fall back to oracle/port.py (the numpy restatement, kind "port").

* reference_gate_timer — pairsim.kernel.apply_gate / apply_controlled_gate
  (kernel.py:108-165) with a pairsim ThreadExecutor (kernel.py:58-89);
* cpu_breadth — per-gate H at n = 20..30 with pairsim's default executor
  (min(cpu, 8) workers, kernel.py:67) and with every host core, QFT(28)
  (config 3) from timed H / cu1 sweeps, config 1, the CPU model;
* paper_harness — the paper's Algorithm 2 through
  pairsim's own harness (bench.py:40-123: BenchConfig, run_benchmark,
  summarize, welch_t_test) with a "b200" back-end registered beside
  pairsim's "engine-parallel".
"""

from __future__ import annotations

import math
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent


def import_pairsim():
    """The unmodified reference package from baseline/_ref, or None."""
    ref = ROOT / "baseline" / "_ref"
    if (ref / "pairsim").is_dir() and str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import pairsim  # noqa: F401
        import pairsim.bench  # noqa: F401
        import pairsim.kernel  # noqa: F401
        import pairsim.measure  # noqa: F401
    except ImportError:
        return None
    return sys.modules["pairsim"]


def cpu_model() -> str:
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform

    return platform.processor() or "unknown"


def host_cores() -> int:
    return len(os.sched_getaffinity(0))


def _avail_bytes() -> int:
    try:
        return os.sysconf("SC_AVPHYS_PAGES") * os.sysconf("SC_PAGE_SIZE")
    except (ValueError, OSError):
        return 0


def fits(n: int) -> bool:
    """pairsim's sweep peaks near 4.5x the register bytes."""
    return 4.6 * (8 << n) <= 0.8 * _avail_bytes()


class ReferenceCPU:
    """One complex64 register on the host and the reference's sweep over it.
    kind "reference" = pairsim itself; "port" = oracle/port.py."""

    def __init__(self, n: int, workers: int | None):
        ps = import_pairsim()
        self.n = n
        if ps is not None:
            from pairsim import gates, kernel, state

            self.kind = "reference"
            self.state = state.new_state(n, memory_budget=1 << 62)
            self.ex = kernel.ThreadExecutor(workers)  # None: pairsim's default min(cpu, 8)
            self.workers = self.ex.workers
            self._g1 = lambda t, g: kernel.apply_gate(self.state, t, g, self.ex)
            self._g2 = lambda c, t, g: kernel.apply_controlled_gate(self.state, c, t, g, self.ex)
            self.H = gates.H
            self.u1 = gates.u1
        else:
            from oracle import port
            from paper_1805_00988_b200.gates import H, u1

            self.kind = "port"
            self.amps = np.zeros(1 << n, np.complex64)
            self.amps[0] = 1
            self.workers = workers or min(os.cpu_count() or 1, 8)
            self.ex = port.Executor(workers=self.workers)
            self._g1 = lambda t, g: port.apply_gate(self.amps, t, g, self.ex)
            self._g2 = lambda c, t, g: port.apply_controlled_gate(self.amps, c, t, g, self.ex)
            self.H = H
            self.u1 = u1

    def h(self, t: int) -> None:
        self._g1(t, self.H)

    def cu1(self, c: int, t: int, theta: float) -> None:
        self._g2(c, t, self.u1(theta))

    def close(self) -> None:
        self.ex.close()

    def describe(self) -> str:
        what = ("pairsim.kernel.apply_gate (unmodified reference from baseline/_ref) with "
                if self.kind == "reference" else "oracle/port.py (numpy restatement of pairsim's sweep) with ")
        return what + f"ThreadExecutor({self.workers} workers)"


def _best(fn, reps: int) -> float:
    best = math.inf
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        best = min(best, time.perf_counter() - t0)
    return best


def cpu_breadth(sizes=(20, 24, 26, 28, 30), budget_s: float = 40.0) -> dict:
    """Per-gate timings of the reference path on this host (best of up to 3
    reps, fewer at large n), both executors; config 3 (QFT(28) = 28 H + 378
    cu1) estimated from its timed H and cu1 sweeps; config 1 timed whole."""
    cores = host_cores()
    out = {"cpu_model": cpu_model(), "host_cores": cores, "per_gate_ms": {}, "executors": {}}
    t_start = time.perf_counter()
    kind = None
    for label, workers in (("default_min_cpu_8", None), ("all_cores", cores)):
        rows = {}
        for n in sizes:
            if not fits(n) or time.perf_counter() - t_start > budget_s:
                rows[str(n)] = None
                continue
            r = ReferenceCPU(n, workers)
            kind = r.kind
            out["executors"][label] = r.workers
            r.h(n // 2)  # warm-up (thread pool, page faults)
            reps = 3 if n <= 26 else 1
            t_h = _best(lambda: r.h(n // 2), reps)
            row = {"h_ms": t_h * 1e3, "GBps": 16 * (1 << n) / t_h / 1e9}
            if n == 28:
                t_c = _best(lambda: r.cu1(n - 1, n // 2, 0.3), reps)
                row["cu1_ms"] = t_c * 1e3
                if label == "all_cores":
                    out["config3_qft28_estimate_s"] = 28 * t_h + 378 * t_c
            rows[str(n)] = row
            r.close()
            del r
        out["per_gate_ms"][label] = rows
    # config 1: 20-qubit H on every qubit + probabilities, whole, all cores
    r = ReferenceCPU(20, cores)

    def config1():
        for q in range(20):
            r.h(q)
        if r.kind == "reference":
            from pairsim import measure

            measure.probabilities(r.state)
        else:
            from oracle import port

            port.probabilities(r.amps)

    config1()
    out["config1_hlayer20_probs_ms"] = _best(config1, 3) * 1e3
    r.close()
    out["kind"] = kind or r.kind
    out["config3_note"] = ("QFT(28) on the CPU = 28 H + 378 cu1 sweeps at n = 28 (circuits.py:195-210), "
                           "estimated from the timed H and cu1 sweeps (a full run takes ~5 min)")
    out["seconds_spent"] = time.perf_counter() - t_start
    return out


def b200_qft_runner(fuse: bool = True):
    """pairsim's engine_qft_runner contract (bench.py:52-69) on the B200:
    allocate the register, run every gate of QFT(n), device barrier (the
    paper times through queue.finish())."""
    from paper_1805_00988_b200 import State, build_qft, execute

    cache: dict = {}

    def run(n: int) -> None:
        circ = cache.get(n) or cache.setdefault(n, build_qft(n))
        s = State(n)
        execute(circ, s, fuse=fuse)
        s.flush()
        s.close()

    return run


def paper_harness(max_qubits: int = 20, samples: int = 6, seed: int = 2018, cpu_max: int = 20,
                  csv_path: str | None = None) -> dict:
    """Algorithm 2 through pairsim's own harness: widths 1..max_qubits, a
    seeded random back-end per trial, one untimed warm-up per (back-end,
    width); Welch's t-test (pairsim.bench.welch_t_test) per width."""
    ps = import_pairsim()
    if ps is None:
        return {"unavailable": "pairsim not installed in baseline/_ref"}
    from pairsim import bench as pb

    from paper_1805_00988_b200 import fusion

    cpu = pb.engine_qft_runner()  # pairsim's threaded engine (default executor)

    def cpu_capped(n: int) -> None:
        if n > cpu_max:
            raise RuntimeError(f"CPU engine skipped above {cpu_max} qubits")
        cpu(n)

    b200 = b200_qft_runner(True)
    for n in range(1, max_qubits + 1):  # queue and finish the pass programs' compiles first
        b200(n)
    fusion.jit_sync()
    cfg = pb.BenchConfig(max_qubits=max_qubits, samples=samples, seed=seed,
                         backends={"b200": b200, "engine-parallel": cpu_capped})
    import warnings

    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        records = pb.run_benchmark(cfg)
    if csv_path:
        pb.write_csv(records, csv_path)
    summ = pb.summarize(records)
    rows = {}
    for n in range(1, max_qubits + 1):
        g = summ.get(("b200", n))
        c = summ.get(("engine-parallel", n))
        row = {"b200_ms": g.mean_seconds * 1e3 if g else None,
               "cpu_ms": c.mean_seconds * 1e3 if c else None}
        if g and c:
            row["speedup"] = c.mean_seconds / g.mean_seconds
            xs = [r.seconds for r in records if r.simulator == "b200" and r.num_qubits == n]
            ys = [r.seconds for r in records if r.simulator == "engine-parallel" and r.num_qubits == n]
            try:
                w = pb.welch_t_test(xs, ys)
                row["welch_t"], row["welch_p"] = w.t, w.p_value
            except Exception as exc:  # InsufficientDataError: too few trials landed here
                row["welch"] = type(exc).__name__
        rows[str(n)] = row
    return {"harness": "pairsim.bench.run_benchmark + welch_t_test (unmodified, baseline/_ref)",
            "backends": ["b200 (fused QFT, State alloc + run + sync)", "engine-parallel (pairsim ThreadExecutor)"],
            "max_qubits": max_qubits, "samples_per_width": samples, "seed": seed, "cpu_max_qubits": cpu_max,
            "records": len(records), "per_width": rows}
