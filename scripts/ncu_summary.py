"""Summarise an `ncu --set full` report into the per-kernel JSON kept under
profiles/ (time, DRAM bytes and rate, IPC, issue / warp activity, registers,
grid, shared-memory bank conflicts).

    python scripts/ncu_summary.py gpurun_out/prof_r01s2.ncu-rep profiles/ncu_full_r01s2_kernels.json [labels...]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "ms": ("gpu__time_duration.sum", 1e-6),
    "dram_read_bytes": ("dram__bytes_read.sum", 1.0),
    "dram_write_bytes": ("dram__bytes_write.sum", 1.0),
    "ipc": ("sm__inst_executed.avg.per_cycle_active", 1.0),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1.0),
    "warps_active_pct": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1.0),
    "registers": ("launch__registers_per_thread", 1.0),
    "grid": ("launch__grid_size", 1.0),
    "smem_bank_conflicts": ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", 1.0),
}
UNIT = {"ms": {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0,
               "s": 1e3, "second": 1e3},
        "bytes": {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}}


def main():
    rep, out = sys.argv[1], sys.argv[2]
    labels = sys.argv[3:]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(head)}
    kernels = []
    for n, r in enumerate(data):
        k = {"kernel": r[col["Kernel Name"]]}
        if n < len(labels):
            k["label"] = labels[n]
        for key, (metric, _) in METRICS.items():
            if metric not in col:
                continue
            v = r[col[metric]].replace(",", "")
            try:
                x = float(v)
            except ValueError:
                continue
            u = units[col[metric]]
            if key == "ms":
                x *= UNIT["ms"].get(u, 1e-6)
            elif key.endswith("_bytes"):
                x *= UNIT["bytes"].get(u, 1.0)
            k[key] = x
        if "ms" in k and "dram_read_bytes" in k and "dram_write_bytes" in k:
            k["dram_GBps"] = round((k["dram_read_bytes"] + k["dram_write_bytes"]) / (k["ms"] * 1e-3) / 1e9, 1)
        kernels.append(k)
    json.dump({"source": rep, "kernels": kernels}, open(out, "w"), indent=1)
    for k in kernels:
        print(k.get("label", ""), k["kernel"][:60], round(k.get("ms", 0), 4), k.get("dram_GBps"))


if __name__ == "__main__":
    main()
