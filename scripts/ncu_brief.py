"""Summarise an ncu --set full capture exported with --page raw --csv (and
optionally --page source --csv --print-source sass): duration, issue / pipe
utilisation, occupancy, stall reasons and the executed instruction mix.

    python scripts/ncu_brief.py RAW.csv [SASS.csv]
"""
from __future__ import annotations

import collections
import csv
import re
import sys

KEYS = [
    ("gpu__time_duration.sum", "duration"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "fma pipe %"),
    ("sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "alu pipe %"),
    ("sm__warps_active.avg.per_cycle_active", "warps/SM"),
    ("smsp__inst_executed.sum", "warp instrs"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("dram__bytes_read.sum", "dram read"),
    ("dram__bytes_write.sum", "dram write"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("smsp__thread_inst_executed_per_inst_executed.ratio", "active lanes/instr"),
]


def raw(path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        d = {h: (v, u) for h, v, u in zip(hdr, vals, units)}
        print(f"== {d.get('Kernel Name', ('?',))[0]}")
        for k, name in KEYS:
            if k in d:
                print(f"  {name:22s} {d[k][0]} {d[k][1]}")
        st = []
        for h, (v, _) in d.items():
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st.append((float(v), h[len("smsp__pcsamp_warps_issue_stalled_"):]))
                except ValueError:
                    pass
        tot = sum(v for v, _ in st) or 1
        print("  stalls: " + ", ".join(f"{n} {100 * v / tot:.1f}%" for v, n in sorted(st, reverse=True)[:9]))


def sass(path):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ci, ie, sc = hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
    cnt, stall, static = collections.Counter(), collections.Counter(), collections.Counter()
    for r in rows[2:]:
        m = re.match(r"(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[ci].strip())
        if not m:
            continue
        op = m.group(2)
        cnt[op] += int(r[ie] or 0)
        stall[op] += int(r[sc] or 0)
        static[op] += 1
    te, ts = sum(cnt.values()) or 1, sum(stall.values()) or 1
    print(f"  static instrs {sum(static.values())}, executed {te}")
    for op, n in cnt.most_common(16):
        print(f"    {op:8s} static {static[op]:5d} exec {100 * n / te:5.1f}% stall {100 * stall[op] / ts:5.1f}%")


if __name__ == "__main__":
    raw(sys.argv[1])
    if len(sys.argv) > 2:
        sass(sys.argv[2])
