#!/usr/bin/env python
"""Benchmark of the gate-sweep hot path (BASELINE.json configs[1]).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Workload (N=1): BASELINE config 2 — a 30-qubit register in HBM, one step =
a Hadamard layer applied as 30 unfused single-qubit sweeps (targets 0..29),
i.e. the per-gate HBM roofline configuration.  metric = single-qubit
gates/s; each sweep moves 16 * 2^30 algorithmic bytes.  The register
(8 GiB) is larger than L2 (126 MB), so no flush is needed between steps.

N>1 (torchrun, one process per GPU): weak scaling — ONE register of
30 + log2(N) qubits sharded over the N GPUs on its top log2(N) qubits
(paper_1805_00988_b200.sharded, NCCL over NVLink).  A step applies H to every
logical qubit; the log2(N) gates on global qubits each trigger a qubit swap
(half-shard NCCL exchange with the partner rank).  value counts shard sweeps
(each 2^30 amplitudes) per second summed over GPUs, so N=1 and N>1 values
are directly comparable.

--impl reference times the reference's own CPU path — pairsim, unmodified,
pip-installed into baseline/_ref (git-ignored, travels to the GPU box;
scripts/refbench.py), its apply_gate with a ThreadExecutor over every host
core — on a bounded sample of the same workload (oracle/port.py, the numpy
restatement, only if baseline/_ref is missing).
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

N_QUBITS = 30
METRIC = "single-qubit gates/sec (H-layer sweep, 30 qubits)"
UNIT = "gates/s"


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--qubits", type=int, default=None)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the fused-pass / config 1, 3, 4 measurements")
    ap.add_argument("--strong", action="store_true",
                    help="strong scaling: a fixed 34-qubit register (--qubits overrides) over the N GPUs; "
                         "reports seconds per H layer and per QFT")
    ap.add_argument("--no-harness", action="store_true", help="skip the paper's Algorithm 2 harness in extras")
    return ap.parse_args()


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# ---------------------------------------------------------------- clocks ----
class ClockSampler:
    """nvidia-smi sampled every 100 ms during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines: list[str] = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, smax, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax = max(smax, float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": smax or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def measured_peak_gbs() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
        except Exception:
            pass
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """dram bytes per sweep launch from the committed ncu --set full capture."""
    for p in sorted((ROOT / "profiles").glob("ncu_sweep_*.json"), reverse=True):
        try:
            return json.loads(p.read_text()).get("dram_bytes_per_launch")
        except Exception:
            continue
    return None


# ------------------------------------------------------------- CPU legs ----
# The reference's own CPU path: pairsim, unmodified, from baseline/_ref
# (scripts/refbench.py); oracle/port.py when that is missing.
CPU_TARGETS = [0, 29, 15, 3, 26, 7, 10, 11, 20, 1, 15, 28, 5, 19, 23, 27, 13, 9]


def cpu_sample(n: int, budget_s: float, threads: int):
    """Time the reference sweep on host cores at the largest n <= the bench's
    that fits host memory.  Returns (gates, seconds, n, ReferenceCPU description, kind)."""
    from scripts.refbench import ReferenceCPU, fits

    while n > 20 and not fits(n):
        n -= 1
    r = ReferenceCPU(n, threads)
    r.h(n // 2)  # warm-up
    t0 = time.perf_counter()
    gates = 0
    while gates < 3 or (time.perf_counter() - t0 < budget_s and gates < len(CPU_TARGETS)):
        r.h(CPU_TARGETS[gates % len(CPU_TARGETS)] % n)
        gates += 1
    dt = time.perf_counter() - t0
    r.close()
    return gates, dt, n, r.describe(), r.kind


def run_reference(args):
    """--impl reference: the reference's CPU implementation of the path
    (pairsim.kernel.apply_gate with a ThreadExecutor over every host core),
    one H sweep of the 30-qubit register per step, targets spread over 0..29
    (stride 11, coprime with 30).  Rank 0 only under torchrun."""
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    from scripts.refbench import ReferenceCPU, cpu_model, fits, host_cores

    threads = host_cores()
    n = args.qubits or N_QUBITS
    while n > 20 and not fits(n):
        n -= 1
    r = ReferenceCPU(n, threads)
    for w in range(args.warmup):
        r.h((w * 11) % n)
    t0 = time.perf_counter()
    for s in range(args.steps):
        r.h(((args.warmup + s) * 11) % n)
    dt = time.perf_counter() - t0
    r.close()
    gates = args.steps
    value = gates / dt
    sample = (f"{gates} H sweeps on a {n}-qubit complex64 register (targets (11 k) mod {n}), "
              f"{r.describe()}, host {cpu_model()} ({threads} cores)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * dt / args.steps,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c64",
        "data": "synthetic", "config": {"workload": "hlayer_sweep", "n_qubits": n, "gates_per_step": 1},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": r.kind, "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }))


# ------------------------------------------------------------- GPU arm ----
def run_ours(args):
    import torch

    rank, world, local = _dist_env()
    if world > 1:
        return run_sharded(args)
    torch.cuda.set_device(local)
    dist = None

    from paper_1805_00988_b200 import State
    from paper_1805_00988_b200.gates import H, m8
    from paper_1805_00988_b200 import _native as N

    n = args.qubits or N_QUBITS
    st = State(n, device=local)
    stream = torch.cuda.ExternalStream(st.stream(), device=torch.device("cuda", local))
    L = N.lib()
    h = st.handle
    hm = m8(H)
    hp = N.f32ptr(hm)

    def layer():
        for t in range(n):
            N.check(L.qs_apply_gate(h, t, hp))

    def barrier():
        torch.cuda.synchronize(local)
        if dist is not None:
            dist.barrier()

    for _ in range(args.warmup):
        layer()
    st.flush()
    barrier()

    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps * n)]
    step_start = torch.cuda.Event(enable_timing=True)
    step_end = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        step_start.record(stream)
        k = 0
        for _ in range(args.steps):
            for t in range(n):
                evs[k][0].record(stream)
                N.check(L.qs_apply_gate(h, t, hp))
                evs[k][1].record(stream)
                k += 1
        step_end.record(stream)
        st.flush()
        barrier()
    total_ms = step_start.elapsed_time(step_end)
    launch_ms = [a.elapsed_time(b) for a, b in evs]
    per_target = [statistics.mean(launch_ms[t::n]) for t in range(n)]
    if dist is not None:
        tt = torch.tensor([total_ms], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        total_ms = float(tt.item())

    gates = args.steps * n * world
    value = gates / (total_ms / 1e3)
    bytes_per_launch = 16 * (1 << n)
    avg_launch_s = statistics.mean(launch_ms) / 1e3
    peak, peak_src = measured_peak_gbs()
    achieved = bytes_per_launch / avg_launch_s / 1e9

    # ---- e2e through the C ABI with pinned host buffers -------------------
    e2e = None
    if not args.no_e2e:
        # Every step uploads a register from pinned host memory, applies the
        # layer and downloads the result.  Two registers are kept in flight so
        # step k+1's H2D overlaps step k's D2H on the other copy engine.
        inp = torch.zeros(2 << n, dtype=torch.float32, pin_memory=True)
        inp[0] = 1.0
        outs = [torch.empty(2 << n, dtype=torch.float32, pin_memory=True) for _ in range(2)]
        st2 = State(n, device=local)
        regs = [st, st2]
        # PCIe-bound (this box: 55-57 GB/s one way, 46 GB/s each way when
        # both directions run, scripts/probes/pcie.py): the first upload and
        # the last download are not overlapped, so a short run under-reports
        # the steady state by (k+1)/k; 20 steps keep that near 5 %.
        k2 = max(20, min(args.steps, 40))

        # the layer as a user runs it: fused passes through qs_apply_fused
        # (compiled pass programs from the second warm-up step on)
        from paper_1805_00988_b200 import build_hadamard_layer, fusion
        from paper_1805_00988_b200.circuits import lower_ops

        layer_passes = fusion.plan(n, lower_ops(build_hadamard_layer(n)))

        def e2e_step(k):
            s = regs[k % 2]
            if k >= 2:
                s.flush()  # its previous step (incl. the download) has finished
            s.upload_async(inp.data_ptr())
            fusion.run(s, layer_passes)
            s.download_async(outs[k % 2].data_ptr())

        for k in range(2):
            e2e_step(k)
        fusion.jit_sync()
        for k in range(2):
            e2e_step(k)
        for s in regs:
            s.flush()
        barrier()
        t0 = time.perf_counter()
        for k in range(k2):
            e2e_step(k)
        for s in regs:
            s.flush()
        barrier()
        dt = time.perf_counter() - t0
        ok = bool(torch.equal(outs[0], outs[1]))
        e2e = {"value": k2 * n * world / dt, "unit": UNIT, "h2d_bytes_per_step": 8 << n,
               "d2h_bytes_per_step": 8 << n, "steps": k2, "outputs_identical": ok,
               "timing": "host wall clock: per step qs_set_amplitudes_async (pinned) + the H layer as "
                         f"{len(layer_passes)} fused passes (qs_apply_fused) + qs_get_amplitudes_async (pinned), "
                         "two registers in flight, synchronized at the end"}
        st2.close()
        del inp, outs
        # the circuit workflow a pairsim user runs (cli `run`: a circuit in,
        # a histogram out): per step the op list goes H2D with the fused
        # passes (kernel parameter blocks), the register starts from |0> on
        # the device (pairsim's new_state), 1000 shots are drawn and the
        # outcomes read back — reported beside e2e, which moves the whole
        # 8 GiB register both ways every step
        try:
            wf = {}
            for mode in ("reset_then_passes", "reset_folded_into_first_pass"):
                folded = mode == "reset_folded_into_first_pass"

                def wf_step(k):
                    if folded:  # execute(measured circuit, initial_basis=0): the first pass writes
                        # |0>'s tiles, the last one leaves the sampler's chunk sums
                        st.sample_prepare(1000)
                        ready = fusion.run(st, layer_passes, from_basis=0, chunk_sums=True)
                        return st.sample_outcomes(1000, k, sums_ready=ready)
                    st.reset(0)
                    fusion.run(st, layer_passes)
                    return st.sample_outcomes(1000, k)

                wf_step(0)
                st.flush()
                reps = 10
                t0 = time.perf_counter()
                for k in range(reps):
                    shots = wf_step(k)
                wf[mode] = reps * n / (time.perf_counter() - t0)
            e2e["circuit_workflow"] = {
                "value": wf["reset_folded_into_first_pass"], "unit": UNIT, "steps": reps,
                "d2h_bytes_per_step": shots.nbytes, "reset_then_passes_value": wf["reset_then_passes"],
                "timing": "host wall clock: |0> + the H layer as fused passes + 1000 exact shots "
                          "(sample_outcomes, int64 outcomes to the host) per step, as execute(measured circuit, "
                          "initial_basis=0) runs it: the reset folded into the first pass, the sampler's chunk "
                          "sums left by the last; reset_then_passes_value = State.reset + passes + sample"}
        except Exception as exc:  # noqa: BLE001
            e2e["circuit_workflow"] = {"error": f"{type(exc).__name__}: {exc}"}

    # extras after e2e: their 8-128 GiB registers and pinned buffers would
    # otherwise precede the PCIe-bound e2e leg in the same process
    extras = {}
    if not args.no_extras and rank == 0:
        extras = run_extras(st, stream, n, cpu=not args.no_cpu, harness=not args.no_harness)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        from scripts.refbench import cpu_breadth, cpu_model, host_cores

        threads = host_cores()
        g, dt, ncpu, desc, kind = cpu_sample(n, 10.0, threads)
        cpu = {"value": g / dt, "unit": UNIT, "cores": threads, "kind": kind, "cpu_model": cpu_model(),
               "sample": f"{g} H sweeps on a {ncpu}-qubit register (targets spread over 0..{ncpu - 1}), "
                         f"{desc}, {dt:.1f} s"}
        try:
            cpu["breadth"] = cpu_breadth()
        except Exception as exc:  # noqa: BLE001
            cpu["breadth"] = {"error": f"{type(exc).__name__}: {exc}"}

    if rank == 0:
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c64", "data": "synthetic",
            "config": {"workload": "hlayer_sweep_unfused", "n_qubits": n, "gates_per_step": n,
                       "state_bytes": 8 << n, "parallelism": f"replicas{world}" if world > 1 else "single",
                       "l2": "register (8 GiB) larger than L2; no flush needed"},
            "gpu_launches": args.steps * n,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": ncu_traffic(),
                         "kernel": "k_sweep_high/k_sweep_low (unfused 1-qubit sweep)",
                         "algorithmic_bytes_per_launch": bytes_per_launch, "peak_source": peak_src,
                         "peak_note": "peak = torch's out-of-place copy_ between two arrays; the sweep "
                                      "reads and writes the same lines in place (likely better DRAM "
                                      "row locality), so it exceeds that copy rate: frac > 1",
                         "frac_of_nominal_8000GBps": achieved / 8000.0,
                         "per_target_ms": [round(x, 4) for x in per_target]},
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if extras:
            out["extras"] = extras
        print(json.dumps(out))
    if dist is not None:
        dist.destroy_process_group()


def run_sharded(args):
    import torch
    import torch.distributed as dist

    from paper_1805_00988_b200 import _native as N
    from paper_1805_00988_b200.gates import H, m8
    from paper_1805_00988_b200.sharded import ShardedState

    rank, world, local = _dist_env()
    local = init_dist()
    g = int(round(math.log2(world)))
    if 1 << g != world:
        raise SystemExit("--gpus must be a power of two")
    L = args.qubits or N_QUBITS
    n = L + g
    # global-target gates: peer gate or NCCL qubit swap + sweep, whichever
    # the calibration on this register measures faster (ShardedState
    # peer_gates="auto"; the global-gate probe below times both)
    st = ShardedState.distributed(n, device=local, peer_gates=os.environ.get("QSB_BENCH_GLOBAL", "auto"))
    eng = st.engines[0]
    stream = torch.cuda.ExternalStream(eng.state.stream(), device=torch.device("cuda", local))

    def layer():
        for q in range(n):
            st.apply_gate(H, q)

    def barrier():
        torch.cuda.synchronize(local)
        dist.barrier()

    for _ in range(args.warmup):
        layer()
    barrier()
    swaps0 = st.swaps
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clocks:
        barrier()
        a.record(stream)
        for _ in range(args.steps):
            layer()
        b.record(stream)
        barrier()
    ms = a.elapsed_time(b)
    tt = torch.tensor([ms], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    ms = float(tt.item())
    swaps = (st.swaps - swaps0) // args.steps
    sweeps = args.steps * n * world
    value = sweeps / (ms / 1e3)

    # roofline of the dominant kernel (the local shard sweep): CUDA events
    # around single local-target sweeps on the shard's stream, max over ranks
    h = eng.state.handle
    hm = m8(H)
    hp = N.f32ptr(hm)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2 * L)]
    barrier()
    for i, (ea, eb) in enumerate(ev):
        ea.record(stream)
        N.check(N.lib().qs_apply_gate(h, i % L, hp))
        eb.record(stream)
    barrier()
    launch_ms = statistics.mean(ea.elapsed_time(eb) for ea, eb in ev)
    tt = torch.tensor([launch_ms], device="cuda")
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    launch_ms = float(tt.item())
    peak, peak_src = measured_peak_gbs()
    bytes_per_launch = 16 * (1 << L)
    achieved = bytes_per_launch / (launch_ms / 1e3) / 1e9
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                "traffic": ncu_traffic() if L == N_QUBITS else None,
                "kernel": "k_sweep_high/k_sweep_low on each rank's shard (local targets)",
                "algorithmic_bytes_per_launch": bytes_per_launch, "peak_source": peak_src,
                "avg_launch_ms": launch_ms, "timing": "CUDA events per launch on the shard stream, "
                                                      "mean over 2 x L local targets, max over ranks"}

    e2e = None
    if not args.no_e2e:
        host = torch.empty(2 << L, dtype=torch.float32, pin_memory=True)
        hptr = host.data_ptr()
        h = eng.state.handle
        L_ = N.lib()
        k2 = max(1, min(args.steps, 2))

        def e2e_step():
            N.check(L_.qs_set_amplitudes(h, 0, 1 << L, hptr))
            layer()
            N.check(L_.qs_get_amplitudes(h, 0, 1 << L, hptr))

        e2e_step()
        barrier()
        t0 = time.perf_counter()
        for _ in range(k2):
            e2e_step()
        barrier()
        dt = time.perf_counter() - t0
        tt = torch.tensor([dt], device="cuda")
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
        e2e = {"value": k2 * n * world / dt, "unit": UNIT, "h2d_bytes_per_step": (8 << L) * world,
               "d2h_bytes_per_step": (8 << L) * world, "steps": k2,
               "timing": "host wall clock, every rank uploads/downloads its shard around the layer, max over ranks"}
    extras = {}
    if not args.no_extras:
        extras["global_gates"] = run_global_gate_probe(n, local, world)
        try:
            eng.state.close()  # the weak-scaling register is done: room for the 34-qubit one
            extras["strong34"] = measure_strong(int(os.environ.get("QSB_BENCH_STRONG_QUBITS", "34")), world, local,
                                                1, 1)
        except Exception as exc:  # noqa: BLE001
            extras["strong34"] = {"error": f"{type(exc).__name__}: {exc}"}
    if not args.no_extras:
        extras["single_process_c_abi"] = run_single_process(n, world, rank)
    if world >= 4 and not args.no_extras:
        extras["config5_hlayer_qft36"] = run_config5(st, eng, local, world)
    line = None
    if rank == 0:
        line = json.dumps({
            "extras": extras,
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "c64", "data": "synthetic",
            "config": {"workload": "hlayer_sweep_unfused_sharded", "n_qubits": n, "shard_qubits": L,
                       "gates_per_step": n, "global_qubit_swaps_per_step": swaps,
                       "global_gate_mode": st.calibration or ("peer" if st.peer_gates else "swap"),
                       "parallelism": f"shard{world} (top {g} qubits)",
                       "value_unit": "shard sweeps (2^%d amplitudes) per second, summed over GPUs" % L,
                       "l2": "shards (8 GiB) larger than L2; no flush needed"},
            "gpu_launches": args.steps * n,
            "roofline": roofline,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "cpu_baseline": None,
        })
    finish_dist(line)


def init_dist() -> int:
    """One rank per GPU over NCCL.  The communicator is created eagerly
    (device_id) with NCCL's INIT-subsystem INFO lines on (rank, nranks, cudaDev
    per communicator) so the logs show every rank joined.  Returns the local
    device."""
    import datetime

    import torch
    import torch.distributed as dist

    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    _, _, local = _dist_env()
    local = local % max(1, torch.cuda.device_count())  # >1 rank per GPU only with QSB_BENCH_SHARE_GPU
    torch.cuda.set_device(local)
    backend = os.environ.get("QSB_BENCH_BACKEND", "nccl")  # gloo: test runs with ranks sharing one GPU
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local),
                                timeout=datetime.timedelta(minutes=10))
    else:
        dist.init_process_group(backend, timeout=datetime.timedelta(minutes=10))
    return local


def finish_dist(line: str | None) -> None:
    """Tear the communicators down on every rank, then let rank 0 print its
    JSON line once no other rank can still write NCCL log lines to the shared
    stdout (a handshake through the launcher's store, which outlives the
    process group)."""
    import torch.distributed as dist

    from torch.distributed import distributed_c10d as c10d

    rank, world, _ = _dist_env()
    store = c10d._get_default_store()
    dist.barrier()
    dist.destroy_process_group()
    sys.stdout.flush()
    store.add("qsb_bench_done", 1)
    if rank == 0:
        deadline = time.time() + 120
        while store.add("qsb_bench_done", 0) < world and time.time() < deadline:
            time.sleep(0.05)
        print(line, flush=True)


def measure_strong(n: int, world: int, local: int, steps: int, warmup: int) -> dict:
    """ONE n-qubit register over the `world` GPUs (world = 1: one device
    register): seconds per H layer (unfused: one sweep per qubit, global
    qubits through qubit swaps), per fused H layer and per QFT(n) (fused
    local passes + swaps, ShardedState.run).  CUDA events on each rank's
    register stream, max over ranks.  Analytic check: QFT (no swaps) maps the
    uniform state to |0>, so after H layer + QFT amplitude 0 must be ~1."""
    import torch

    from paper_1805_00988_b200 import _native as N
    from paper_1805_00988_b200 import build_hadamard_layer, build_qft, fusion
    from paper_1805_00988_b200.gates import H
    from paper_1805_00988_b200.sharded import ShardedState

    g = int(round(math.log2(world)))
    N.lib().qs_release_cached(-1)
    free_b, _ = torch.cuda.mem_get_info(local)
    budget = max(1, free_b - (6 << 30))
    if world > 1:
        st = ShardedState.distributed(n, device=local, memory_budget=budget)
    else:
        st = ShardedState.virtual(n, 1, device=local, memory_budget=budget)
    eng = st.engines[0]
    stream = torch.cuda.ExternalStream(eng.state.stream(), device=torch.device("cuda", local))

    def barrier():
        torch.cuda.synchronize(local)
        if world > 1:
            import torch.distributed as dist

            dist.barrier()

    def timed(fn, reps):
        barrier()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(reps):
            fn()
        b.record(stream)
        barrier()
        return a.elapsed_time(b) / 1e3 / reps

    def layer():
        for q in range(n):
            st.apply_gate(H, q)

    hl, qft = build_hadamard_layer(n), build_qft(n)
    for _ in range(warmup):
        layer()
    swaps0 = st.swaps
    t_layer = timed(layer, steps)
    swaps = (st.swaps - swaps0) / steps
    st.run(hl)
    st.run(qft)  # queues the pass programs' compiles
    fusion.jit_sync()
    st.reset(0)
    t_fused = timed(lambda: st.run(hl), 1)
    t_qft = timed(lambda: st.run(qft), 1)
    st.run(qft, exact=False)  # compiles of the inexact programs
    fusion.jit_sync()
    st.reset(0)
    st.run(hl)
    t_qft_inexact = timed(lambda: st.run(qft, exact=False), 1)
    st.reset(0)
    st.run(hl)
    st.run(qft)  # the exact result again for the analytic check below
    vals = [t_layer, t_fused, t_qft, t_qft_inexact]
    if world > 1:
        import torch.distributed as dist

        t = torch.tensor(vals, device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        vals = [float(x) for x in t.tolist()]
    st.canonicalize()
    a0 = complex(eng.state.amplitude(0)) if st.ranks[0] == 0 else None
    out = {"n_qubits": n, "n_gpus": world, "shard_qubits": n - g, "hlayer_s": vals[0], "hlayer_fused_s": vals[1],
           "qft_s": vals[2], "qft_inexact_s": vals[3], "qft_gates": qft.gate_count(),
           "global_qubit_swaps_per_layer": swaps,
           "timing": "CUDA events on each rank's register stream, max over ranks"}
    if a0 is not None:
        out["amp0_after_hlayer_qft"] = [a0.real, a0.imag]
        out["analytic_check_ok"] = bool(abs(a0 - 1.0) < 1e-3)
    st.close()
    N.lib().qs_release_cached(-1)
    return out


def run_strong(args):
    """--strong: the strong-scaling line (SURVEY 8(e) "Reporting"), value =
    seconds per unfused H layer of ONE 34-qubit register (--qubits
    overrides) over the N GPUs; the fused layer and QFT(n) ride along."""
    import torch

    rank, world, local = _dist_env()
    n = args.qubits or 34
    if world > 1:
        local = init_dist()
    else:
        torch.cuda.set_device(local)
    with ClockSampler(local) as clocks:
        r = measure_strong(n, world, local, args.steps, args.warmup)
    line = json.dumps({
        "metric": f"seconds per H layer ({n} qubits, strong scaling)", "value": r["hlayer_s"], "unit": "s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["hlayer_s"] * 1e3,
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None, "dtype": "c64", "data": "synthetic",
        "config": {"workload": f"hlayer{n}_strong", "n_qubits": n, "shard_qubits": r["shard_qubits"],
                   "parallelism": f"shard{world}" if world > 1 else "single",
                   "global_qubit_swaps_per_layer": r["global_qubit_swaps_per_layer"]},
        "strong": r, "gpu_launches": args.steps * n, "clocks": clocks.summary(),
    })
    if world > 1:
        finish_dist(line if rank == 0 else None)
    else:
        print(line)


def run_single_process(n, world, rank):
    """The same register driven by ONE process over all N GPUs through the C
    ABI (qs_create_sharded: ncclCommInitAll communicators, NCCL or peer
    exchanges).  Rank 0 runs it while the other ranks wait at a barrier.
    Host wall clock around device-synchronised calls."""
    import torch.distributed as dist

    out = None
    if rank == 0:
        try:
            from paper_1805_00988_b200 import build_qft, fusion
            from paper_1805_00988_b200.multigpu import MultiDeviceState

            out = {"n_qubits": n, "devices": world}
            for label, exch, peer in (("nccl_swaps", "nccl", False), ("p2p_swaps", "p2p", False),
                                      ("peer_gates", "p2p", True)):
                import torch

                md = MultiDeviceState(n, [r % torch.cuda.device_count() for r in range(world)])
                try:
                    md.set_mode(peer_gates=peer, exchange=exch)
                except Exception as exc:  # noqa: BLE001  (e.g. no NCCL communicators)
                    out[label] = {"error": f"{type(exc).__name__}: {exc}"}
                    md.close()
                    continue
                for q in range(n):
                    md.h(q)
                md.flush()
                md.reset(0)
                md.flush()
                t0 = time.perf_counter()
                for q in range(n):
                    md.h(q)
                md.flush()
                t_layer = time.perf_counter() - t0
                t0 = time.perf_counter()
                md.run(build_qft(n), fuse=False)
                md.flush()
                t_qft = time.perf_counter() - t0
                md.run(build_qft(n))  # fused local passes: compiles, then timed
                fusion.jit_sync()
                md.flush()
                t0 = time.perf_counter()
                md.run(build_qft(n))
                md.flush()
                t_qft_f = time.perf_counter() - t0
                out[label] = {"hlayer_ms": t_layer * 1e3, "qft_unfused_ms": t_qft * 1e3,
                              "qft_fused_ms": t_qft_f * 1e3, **md.stats()}
                md.close()
            if world >= 4:  # config 5 through the single-process C ABI
                out["config5_hlayer_qft36"] = _config5_single_process(world)
            from paper_1805_00988_b200 import _native as N

            N.lib().qs_release_cached(-1)  # hand the other ranks' devices their memory back
        except Exception as exc:  # noqa: BLE001
            out = {"error": f"{type(exc).__name__}: {exc}"}
    dist.barrier()
    return out


def _config5_single_process(world):
    """BASELINE config 5 driven by one process (qs_create_sharded over the N
    devices): H on all 36 qubits, then QFT(36) with fused local passes;
    analytic check |amplitude(0)| ~ 1."""
    try:
        import torch

        from paper_1805_00988_b200 import _native as N
        from paper_1805_00988_b200 import build_hadamard_layer, build_qft, fusion
        from paper_1805_00988_b200.multigpu import MultiDeviceState

        N.lib().qs_release_cached(-1)
        ndev = torch.cuda.device_count()
        free_b = min(torch.cuda.mem_get_info(d)[0] for d in range(ndev))
        md = MultiDeviceState(36, [r % ndev for r in range(world)], memory_budget=max(1, free_b - (6 << 30)))
        try:
            md.run(build_hadamard_layer(36))
            md.run(build_qft(36))
            fusion.jit_sync()
            md.reset(0)
            md.flush()
            t0 = time.perf_counter()
            md.run(build_hadamard_layer(36))
            md.flush()
            t1 = time.perf_counter()
            md.run(build_qft(36))
            md.flush()
            t2 = time.perf_counter()
            a0 = complex(md.amplitudes(0, 1)[0])
            return {"hlayer_s": t1 - t0, "qft_s": t2 - t1, **md.stats(), "amp0_after_qft": [a0.real, a0.imag],
                    "analytic_check_ok": bool(abs(abs(a0) - 1.0) < 1e-2), "timing": "host wall clock, synchronised"}
        finally:
            md.close()
    except Exception as exc:  # noqa: BLE001
        return {"error": f"{type(exc).__name__}: {exc}"}


def run_global_gate_probe(n, local, world, reps=3):
    """H on each of the log2(N) global qubits from the identity qubit map:
    NCCL qubit swaps + local sweeps (default path) vs one peer-memory kernel
    per partner pair over NVLink (csrc/peer.cu).  Host wall clock between
    device-synchronised barriers, max over ranks."""
    import torch
    import torch.distributed as dist

    from paper_1805_00988_b200.gates import H
    from paper_1805_00988_b200.sharded import ShardedState

    g = int(round(math.log2(world)))
    out = {"n_qubits": n, "global_qubits": g}
    for name, peer in (("swap_nccl", False), ("peer_nvlink", True), ("auto_calibrated", "auto")):
        try:
            st = ShardedState.distributed(n, device=local, peer_gates=peer)
            best = float("inf")
            for _ in range(reps + 1):
                st.reset(0)
                st.synchronize()
                torch.cuda.synchronize(local)
                dist.barrier()
                t0 = time.perf_counter()
                for q in range(n - g, n):
                    st.apply_gate(H, q)
                st.synchronize()
                torch.cuda.synchronize(local)
                dist.barrier()
                best = min(best, time.perf_counter() - t0)
            t = torch.tensor([best], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            out[name] = {"ms_per_global_gate": float(t.item()) * 1e3 / g,
                         "swaps_per_rep": st.swaps // (reps + 1),
                         "peer_gates_per_rep": st.peer_gate_count // (reps + 1),
                         "peer_mode_active": st.peer_gates, "calibration": st.calibration}
            del st
        except Exception as exc:  # noqa: BLE001
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
    return out


def run_config5(st_main, eng_main, local, world):
    """BASELINE config 5: a 36-qubit register sharded over the N GPUs (top
    log2 N qubits), H on every qubit then build_qft(36), through
    ShardedState.run (fused local passes + NCCL qubit swaps).  Device time on
    every rank's stream, max over ranks.  Analytic check: QFT (no swaps) of the
    uniform state is |0>, so amplitude 0 must be ~1."""
    import torch
    import torch.distributed as dist

    from paper_1805_00988_b200 import _native as N
    from paper_1805_00988_b200 import build_hadamard_layer, build_qft
    from paper_1805_00988_b200.sharded import ShardedState

    n = 36
    out = {"n_qubits": n, "shards": world}
    try:
        # free the headline registers (and the pool's cached buffers) first
        eng_main.state.close()
        N.lib().qs_release_cached(-1)
        torch.cuda.synchronize(local)
        # a 36-qubit register on 4 GPUs is a 128 GiB shard: above the default
        # 75%-of-free budget, so budget all but 6 GiB of the free memory
        free_b, _ = torch.cuda.mem_get_info(local)
        st, why = None, ""
        try:
            st = ShardedState.distributed(n, device=local, memory_budget=max(1, free_b - (6 << 30)))
        except Exception as exc:  # noqa: BLE001
            why = f"{type(exc).__name__}: {exc}"
        ok = torch.tensor([1 if st is not None else 0], device="cuda")
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)  # every rank allocated, or none proceeds
        if int(ok.item()) != 1:
            out["error"] = "allocation failed on a rank" + (f": {why}" if why else "")
            return out
        eng = st.engines[0]
        stream = torch.cuda.ExternalStream(eng.state.stream(), device=torch.device("cuda", local))
        torch.cuda.synchronize(local)
        dist.barrier()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        evs[0].record(stream)
        st.run(build_hadamard_layer(n))
        evs[1].record(stream)
        st.run(build_qft(n))
        evs[2].record(stream)
        torch.cuda.synchronize(local)
        dist.barrier()
        t = torch.tensor([evs[0].elapsed_time(evs[1]), evs[1].elapsed_time(evs[2])], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        h_ms, q_ms = (float(x) for x in t.tolist())
        swaps = st.swaps
        a0 = None
        st.canonicalize()  # identity qubit map, so amplitude 0 is rank 0's first
        if st.ranks[0] == 0:
            a0 = complex(eng.state.amplitude(0))
        out.update({"hlayer_s": h_ms / 1e3, "qft_s": q_ms / 1e3, "total_s": (h_ms + q_ms) / 1e3,
                    "qft_gates": build_qft(n).gate_count(), "global_qubit_swaps": swaps,
                    "shard_bytes": 8 << (n - int(math.log2(world)))})
        if a0 is not None:
            out["amp0_after_qft"] = [a0.real, a0.imag]
            out["analytic_check_ok"] = bool(abs(abs(a0) - 1.0) < 1e-2)
    except Exception as exc:  # noqa: BLE001
        out["error"] = f"{type(exc).__name__}: {exc}"
    return out


def run_extras(st, stream, n, cpu=True, harness=True):
    """Fused passes on the 30-qubit register, plus BASELINE configs 1, 3, 4."""
    import torch

    from paper_1805_00988_b200 import State, build_hadamard_layer, build_qft, fusion, layered_random_circuit
    from paper_1805_00988_b200.circuits import lower_ops

    def timed(state, strm, passes, reps=3, combine=False, cold=None):
        # first run = the cold number (pass programs' compiles queued on host
        # threads, csrc/jit.cu, the passes meanwhile on the interpreter
        # kernel); then wait for the compiles so the timed runs launch
        # compiled programs only
        t0 = time.perf_counter()
        fusion.run(state, passes, combine=combine)
        state.flush()
        if cold is not None:
            cold.append((time.perf_counter() - t0) * 1e3)
        fusion.jit_sync()
        fusion.run(state, passes, combine=combine)
        state.flush()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(strm)
        for _ in range(reps):
            fusion.run(state, passes, combine=combine)
        b.record(strm)
        state.flush()
        return a.elapsed_time(b) / reps

    def fused_entry(circ, nq, state, strm, exact=True, reps=3):
        passes = fusion.plan(nq, lower_ops(circ), reorder=not exact)
        cold = []
        ms = timed(state, strm, passes, reps=reps, combine=not exact, cold=cold)
        return {"gates": circ.gate_count(), "passes": len(passes), "ms": ms, "cold_first_run_ms": cold[0],
                "jit_programs_so_far": fusion.jit_stats(),
                "effective_gates_per_s": circ.gate_count() / (ms / 1e3),
                "pass_bytes": len(passes) * 16 * (1 << nq),
                "achieved_GBps": len(passes) * 16 * (1 << nq) / (ms / 1e3) / 1e9,
                "mode": "exact (bit-identical to the reference)" if exact else
                        "exact=False (reordered passes + combined diagonal runs; rtol 1e-5 vs the reference)"}

    res = {}
    res["hlayer30_fused"] = fused_entry(build_hadamard_layer(n), n, st, stream)
    res["qft30_fused"] = fused_entry(build_qft(n), n, st, stream)
    res["qft30_fused_inexact"] = fused_entry(build_qft(n), n, st, stream, exact=False)

    # K2 / K3 / K4 single-op sweeps at full size (touched bytes
    # and the full-sweep equivalent reported separately)
    from paper_1805_00988_b200 import random_unitary_gate, u1 as _u1
    import numpy as _np

    g = random_unitary_gate(_np.random.default_rng(5))
    kern = {}
    for name, fn, touched in (
            ("controlled_c29_t7", lambda: st.apply_controlled_gate(g, n - 1, 7), 8 << n),
            ("controlled_c0_t7", lambda: st.apply_controlled_gate(g, 0, 7), 8 << n),
            ("controlled_c3_t1", lambda: st.apply_controlled_gate(g, 3, 1), 8 << n),
            ("ccontrolled_c29_c28_t7", lambda: st.apply_controlled_controlled_gate(g, n - 1, n - 2, 7), 4 << n),
            ("cphase_c29_t7", lambda: st.apply_controlled_gate(_u1(0.3), n - 1, 7), 4 << n)):
        fn()
        st.flush()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(5):
            fn()
        b.record(stream)
        st.flush()
        ms = a.elapsed_time(b) / 5
        kern[name] = {"ms": round(ms, 4), "touched_GBps": round(touched / ms / 1e6, 1),
                      "full_sweep_equiv_GBps": round((16 << n) / ms / 1e6, 1)}
    res["single_op_kernels30"] = kern

    # config 1: 20-qubit H on every qubit + probabilities (host wall clock, incl. the fp64 D2H)
    s20 = State(20)
    s20.h(0)
    s20.probabilities()
    best = float("inf")
    for _ in range(5):
        t0 = time.perf_counter()
        s20.reset(0)
        for q in range(20):
            s20.h(q)
        probs = s20.probabilities()
        best = min(best, time.perf_counter() - t0)
    res["config1_hlayer20_probs"] = {"ms_wall": best * 1e3, "gates": 20,
                                     "note": "State(20).reset + 20 x h + probabilities() to host, best of 5"}
    if cpu:
        from scripts.refbench import ReferenceCPU, host_cores

        r = ReferenceCPU(20, host_cores())
        cbest = float("inf")
        for _ in range(3):
            t0 = time.perf_counter()
            if r.kind == "reference":
                r.state.amps[:] = 0
                r.state.amps[0] = 1
            else:
                r.amps[:] = 0
                r.amps[0] = 1
            for q in range(20):
                r.h(q)
            if r.kind == "reference":
                from pairsim import measure as _pm

                p = _pm.probabilities(r.state)
            else:
                from oracle import port

                p = port.probabilities(r.amps)
            cbest = min(cbest, time.perf_counter() - t0)
        r.close()
        res["config1_hlayer20_probs"]["cpu_ms"] = cbest * 1e3
        res["config1_hlayer20_probs"]["cpu_kind"] = r.kind
        res["config1_hlayer20_probs"]["probabilities_bit_identical"] = bool(p.tobytes() == probs.tobytes())
    s20.close()

    # launch-bound small registers: QFT(16) as 136 separate sweeps, launched
    # from Python one by one vs recorded once into a CUDA graph and replayed
    from paper_1805_00988_b200 import execute

    s16 = State(16)
    s16_stream = torch.cuda.ExternalStream(s16.stream())
    q16 = build_qft(16)
    execute(q16, s16, fuse=False)
    s16.flush()
    t0 = time.perf_counter()
    for _ in range(10):
        execute(q16, s16, fuse=False)
    s16.flush()
    direct_ms = (time.perf_counter() - t0) * 1e3 / 10
    with s16.record() as rec:
        execute(q16, s16, fuse=False)
    rec.graph.replay(1)
    s16.flush()
    t0 = time.perf_counter()
    rec.graph.replay(10)
    s16.flush()
    graph_ms = (time.perf_counter() - t0) * 1e3 / 10
    rec.graph.close()
    s16.close()
    res["graph_qft16_unfused"] = {"gates": q16.gate_count(), "direct_ms": direct_ms, "graph_replay_ms": graph_ms,
                                  "note": "host wall clock per circuit, 10 reps; direct = one ctypes call + "
                                          "launch per gate, graph = State.record() once, Graph.replay()"}

    # measure path on the 30-qubit register: the exact sampling chain (M1-M6,
    # device-only; cost depends on the state's CDF) on a generic state, the
    # uniform state and a basis state, and probabilities to the host into a
    # fresh pageable array (first touch included) and into a reused pinned one
    from paper_1805_00988_b200 import _native as _Nm

    samp = {}
    for kind in ("generic", "uniform", "basis"):
        if kind == "uniform":
            st.reset(0)
            for q in range(n):
                st.h(q)
        elif kind == "basis":
            st.reset(123456789)
        st.sample_outcomes(1_000_000, 1)  # warm: scratch and pinned result buffers sized for 10^6 draws
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(stream)
        st.sample_outcomes(1_000_000, 2)
        b.record(stream)
        st.flush()
        samp[kind] = a.elapsed_time(b)
    st.reset(0)
    for q in range(n):
        st.h(q)
    st.t(3)
    st.flush()  # the gates above are asynchronous: not part of the readout
    t0 = time.perf_counter()
    pr = st.probabilities()
    t_first = time.perf_counter() - t0  # incl. the staging buffers' first allocation
    del pr
    t_pr = 1e9
    for _ in range(2):  # a fresh result array each call (page faults included)
        t0 = time.perf_counter()
        pr = st.probabilities()
        t_pr = min(t_pr, time.perf_counter() - t0)
        del pr
    pin = _Nm.pinned_empty(1 << n)
    st.probabilities(out=pin)
    t0 = time.perf_counter()
    st.probabilities(out=pin)
    t_pin = time.perf_counter() - t0
    res["measure30"] = {"sample_1e6_ms": samp, "probabilities_to_host_ms": t_pr * 1e3,
                        "probabilities_to_host_first_call_ms": t_first * 1e3,
                        "probabilities_to_pinned_ms": t_pin * 1e3,
                        "probabilities_bytes": 8 << n,
                        "probabilities_GBps": {"fresh_pageable": (8 << n) / t_pr / 1e9,
                                               "reused_pinned": (8 << n) / t_pin / 1e9},
                        "note": "sample: exact sequential-CDF chain + 1e6 PCG64 draws (bit-exact with "
                                "pairsim.sample), CUDA events, per state kind (generic = after the fused "
                                "circuits above, uniform = H layer, basis = |123456789>); probabilities: fp64 "
                                "|a|^2 to a fresh numpy array (staged through pinned buffers, page faults "
                                "included) and into a reused pinned array (State.probabilities(out=...), "
                                "direct DMA), host wall clock"}
    del pin

    # config 3: 28-qubit QFT (fused), parity vs pairsim is in tests/test_gpu_parity.py
    s28 = State(28)
    s28_stream = torch.cuda.ExternalStream(s28.stream())
    res["config3_qft28_fused"] = fused_entry(build_qft(28), 28, s28, s28_stream)
    res["config3_qft28_fused_inexact"] = fused_entry(build_qft(28), 28, s28, s28_stream, exact=False)
    s28.close()

    # complex128 (Precision.DOUBLE) sweeps: a 29-qubit register is 8 GiB like
    # the headline one; each sweep moves 32 * 2^29 algorithmic bytes
    from paper_1805_00988_b200.gates import H as _H

    sd = State(29, precision="double")
    sd_stream = torch.cuda.ExternalStream(sd.stream())
    for q in range(29):
        sd.apply_gate(_H, q)
    sd.flush()
    per = []
    for q in range(29):
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(sd_stream)
        for _ in range(3):
            sd.apply_gate(_H, q)
        b.record(sd_stream)
        sd.flush()
        per.append(a.elapsed_time(b) / 3)
    avg = sum(per) / len(per)
    # complex128 QFT(28) (4 GiB) as compiled TMA tile passes vs one sweep per gate
    sq = State(28, precision="double")
    sq_stream = torch.cuda.ExternalStream(sq.stream())
    q28 = build_qft(28)
    dpasses = fusion.plan(28, lower_ops(q28, double=True), 12)
    ms_f = timed(sq, sq_stream, dpasses, reps=2)
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    from paper_1805_00988_b200 import execute as _ex

    a.record(sq_stream)
    _ex(q28, sq, fuse=False)
    b.record(sq_stream)
    sq.flush()
    res["c128_qft28"] = {"gates": q28.gate_count(), "passes": len(dpasses), "fused_ms": ms_f,
                         "unfused_ms": a.elapsed_time(b),
                         "note": "complex128 register; fused = compiled TMA tile programs (16-B one-amplitude units)"}
    sq.close()
    res["c128_hsweep29"] = {"ms_per_sweep_avg": avg, "ms_per_target": [round(x, 4) for x in per],
                            "algorithmic_bytes_per_sweep": 32 << 29,
                            "achieved_GBps": (32 << 29) / (avg / 1e3) / 1e9,
                            "note": "complex128 register (8 GiB), H on every target, 3 reps each, CUDA events"}
    sd.close()

    # the sharded machinery at full size on one GPU: a 31-qubit register as 2
    # virtual shards of 30 qubits (16 GiB), H on every qubit; the global qubit
    # goes through a qubit swap (in-process D2D exchange) or the peer-memory
    # kernel (partner shard in the same HBM standing in for an NVLink peer)
    from paper_1805_00988_b200.sharded import ShardedState
    from paper_1805_00988_b200.gates import H as _Hg

    from paper_1805_00988_b200 import _native as _N

    sv = {}
    for mode, peer, exch in (("swap_copy", False, "nccl"), ("swap_peer_kernel", False, "peer"),
                             ("peer_gates", True, "peer")):
        vs = ShardedState.virtual(31, 2, peer_gates=peer, exchange=exch)
        for q in range(31):
            vs.apply_gate(_Hg, q)
        vs.synchronize()
        vs.reset(0)
        vs.synchronize()
        t0 = time.perf_counter()
        for q in range(31):
            vs.apply_gate(_Hg, q)
        vs.synchronize()
        sv[mode] = {"layer_ms": (time.perf_counter() - t0) * 1e3, "swaps": vs.swaps,
                    "peer_gates": vs.peer_gate_count}
        vs.close()
        _N.lib().qs_release_cached(-1)
    # the exchange alone (data movement of one qubit swap: each of the two
    # 30-qubit shards trades half its amplitudes, 2 x 4 GiB) against a D2D
    # copy of the same 8 GiB (>= 0.8 of the copy rate)
    try:
        xs = {}
        payload = 2 * (1 << 29) * 8
        for mode, exch in (("copy_exchange", "nccl"), ("peer_swap_kernel", "peer")):
            vs = ShardedState.virtual(31, 2, peer_gates=False, exchange=exch)
            vs._exchange(0)
            vs.synchronize()
            reps = 4
            t0 = time.perf_counter()
            for _ in range(reps):
                vs._exchange(0)
            vs.synchronize()
            dt = (time.perf_counter() - t0) / reps
            xs[mode] = {"ms": dt * 1e3, "payload_GBps": payload / dt / 1e9}
            vs.close()
            _N.lib().qs_release_cached(-1)
        src_t = torch.empty(payload // 4, dtype=torch.float32, device="cuda")
        dst_t = torch.empty_like(src_t)
        dst_t.copy_(src_t)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(4):
            dst_t.copy_(src_t)
        torch.cuda.synchronize()
        dt = (time.perf_counter() - t0) / 4
        xs["d2d_copy_same_payload"] = {"ms": dt * 1e3, "payload_GBps": payload / dt / 1e9}
        for mode in ("copy_exchange", "peer_swap_kernel"):
            xs[mode]["vs_d2d_copy"] = xs["d2d_copy_same_payload"]["ms"] / xs[mode]["ms"]
        del src_t, dst_t
        sv["exchange_alone"] = {**xs, "note": "host wall clock per exchange (synchronized), 4 reps; payload = "
                                              "the 8 GiB that change shards"}
    except Exception as exc:  # noqa: BLE001
        sv["exchange_alone"] = {"error": f"{type(exc).__name__}: {exc}"}
    # the same layer through the single-process C ABI (qs_create_sharded)
    from paper_1805_00988_b200.multigpu import MultiDeviceState

    for mode, peer in (("c_abi_swap", False), ("c_abi_peer_gates", True)):
        md = MultiDeviceState(31, [0, 0], peer_gates=peer)
        for q in range(31):
            md.h(q)
        md.flush()
        md.reset(0)
        md.flush()
        t0 = time.perf_counter()
        for q in range(31):
            md.h(q)
        md.flush()
        sv[mode] = {"layer_ms": (time.perf_counter() - t0) * 1e3, **md.stats()}
        md.close()
        _N.lib().qs_release_cached(-1)
    res["sharded_virtual_31q_2shards"] = {**sv, "note": "H layer over 31 qubits as 2 virtual shards on one "
                                          "B200 (host wall clock incl. per-gate syncs of the sharded layer)"}

    # config 5's machinery at its per-GPU shard size on one GPU: a 33-qubit
    # register as 8 virtual 30-qubit shards (64 GiB), H on every qubit then
    # build_qft(33) through ShardedState.run (fused local passes per shard,
    # 3 global qubits, qubit swaps in HBM standing in for NVLink); analytic
    # check as in config 5 (QFT of the uniform state is |0>)
    try:
        from paper_1805_00988_b200 import build_hadamard_layer as _bhl, build_qft as _bqft

        n5 = 33
        v5 = ShardedState.virtual(n5, 8)
        v5.synchronize()
        t0 = time.perf_counter()
        v5.run(_bhl(n5))
        v5.synchronize()
        t1 = time.perf_counter()
        v5.run(_bqft(n5))
        v5.synchronize()
        t2 = time.perf_counter()
        sw = v5.swaps
        v5.canonicalize()
        a0 = complex(v5.engines[0].state.amplitude(0))
        res["config5_machinery_virtual_33q_8shards"] = {
            "hlayer_s": t1 - t0, "qft_s": t2 - t1, "qft_gates": _bqft(n5).gate_count(), "global_qubit_swaps": sw,
            "amp0_after_qft": [a0.real, a0.imag], "analytic_check_ok": bool(abs(abs(a0) - 1.0) < 1e-2),
            "note": "8 virtual 30-qubit shards on one B200 (host wall clock, exchanges are in-HBM copies): "
                    "the config-5 code path at its per-GPU shard size, not an NVLink number"}
        v5.close()
        _N.lib().qs_release_cached(-1)
    except Exception as exc:  # noqa: BLE001
        res["config5_machinery_virtual_33q_8shards"] = {"error": f"{type(exc).__name__}: {exc}"}

    # per-gate H sweeps at the CPU baseline's sizes (cpu_baseline.breadth)
    per_n = {}
    for nn in (20, 24, 26, 28):
        sn = State(nn)
        sn_stream = torch.cuda.ExternalStream(sn.stream())
        for q in range(nn):
            sn.h(q)
        sn.flush()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        a.record(sn_stream)
        for rep in range(5):
            for q in range(nn):
                sn.h(q)
        b.record(sn_stream)
        sn.flush()
        ms = a.elapsed_time(b) / (5 * nn)
        per_n[str(nn)] = {"h_ms": ms, "GBps": 16 * (1 << nn) / ms / 1e6}
        sn.close()
    per_n["30"] = {"h_ms": None, "note": "the headline (roofline.per_target_ms)"}
    res["per_gate_by_n"] = {**per_n, "note": "H on every target, 5 layers, CUDA events; n <= 24 fits L2"}

    if harness:
        try:
            from scripts.refbench import paper_harness

            res["paper_algorithm2"] = paper_harness(max_qubits=20, samples=6)
        except Exception as exc:  # noqa: BLE001
            res["paper_algorithm2"] = {"error": f"{type(exc).__name__}: {exc}"}

    # config 4: 32-qubit layered random H/T/CX circuit, depth 20, fused
    try:
        s32 = State(32)
    except Exception as exc:  # noqa: BLE001
        res["config4_random32_fused"] = {"skipped": str(exc)}
        return res
    s32_stream = torch.cuda.ExternalStream(s32.stream())
    circ = layered_random_circuit(32, 20, seed=32)
    res["config4_random32_fused"] = fused_entry(circ, 32, s32, s32_stream, reps=1)
    try:
        s32b = State(32)
        s32b_stream = torch.cuda.ExternalStream(s32b.stream())
        ent = fused_entry(circ, 32, s32b, s32b_stream, exact=False, reps=1)
        # agreement with the exact result (both registers hold the circuit
        # applied to the previous contents: reset and run once more each)
        for s_, ex in ((s32, True), (s32b, False)):
            s_.reset(0)
            fusion.run(s_, fusion.plan(32, lower_ops(circ), reorder=not ex), combine=not ex)
            s_.flush()

        def tview(s_):
            ptr, nf = s_.device_pointer(), 2 << 32

            class _CAI:
                __cuda_array_interface__ = {"shape": (nf,), "typestr": "<f4", "data": (ptr, False),
                                            "version": 3, "strides": None}

            return torch.as_tensor(_CAI(), device=torch.device("cuda", torch.cuda.current_device()))

        va, vb = tview(s32), tview(s32b)
        worst, peak = 0.0, 0.0
        for off in range(0, va.numel(), 1 << 28):
            worst = max(worst, float((va[off: off + (1 << 28)] - vb[off: off + (1 << 28)]).abs().max()))
            peak = max(peak, float(va[off: off + (1 << 28)].abs().max()))
        ent["max_abs_diff_vs_exact"] = worst
        ent["max_abs_amplitude"] = peak
        res["config4_random32_fused_inexact"] = ent
        del va, vb
        s32b.close()
    except Exception as exc:  # noqa: BLE001
        res["config4_random32_fused_inexact"] = {"error": f"{type(exc).__name__}: {exc}"}
    s32.close()

    # strong-scaling reference point: one 34-qubit register (128 GiB) on this GPU
    try:
        res["strong34"] = measure_strong(34, 1, torch.cuda.current_device(), 1, 1)
    except Exception as exc:  # noqa: BLE001
        res["strong34"] = {"error": f"{type(exc).__name__}: {exc}"}
    return res


def _free_port() -> int:
    import socket

    with socket.socket() as sock:
        sock.bind(("127.0.0.1", 0))
        return sock.getsockname()[1]


def _visible_gpus() -> int:
    import torch

    return torch.cuda.device_count()


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
        return
    world_env = os.environ.get("WORLD_SIZE")
    if world_env is None and args.gpus > 1:
        # `python bench.py --gpus N` without a launcher: start N ranks (one
        # process per GPU) under torch.distributed.run ourselves
        have = _visible_gpus()
        if have < args.gpus and os.environ.get("QSB_BENCH_SHARE_GPU") != "1":
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but only {have} GPU(s) are visible\n")
            sys.exit(2)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr=127.0.0.1", f"--master-port={_free_port()}", str(Path(__file__).resolve()),
               *sys.argv[1:]]
        sys.exit(subprocess.call(cmd))
    world = int(world_env or 1)
    if world != args.gpus:
        sys.stderr.write(f"bench.py: WORLD_SIZE={world} but --gpus {args.gpus}\n")
        sys.exit(2)
    if world > 1 and _visible_gpus() < world and os.environ.get("QSB_BENCH_SHARE_GPU") != "1":
        sys.stderr.write(f"bench.py: {world} ranks but only {_visible_gpus()} GPU(s) are visible\n")
        sys.exit(2)
    if args.strong:
        run_strong(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
