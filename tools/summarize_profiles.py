"""Summaries of ncu output for profiles/ (run in the dev container).

    # launch list of a short bench run (per-launch durations, cold, serialized)
    python tools/summarize_profiles.py launches gpurun_out/launches.csv > profiles/rXX_launches_summary.txt
    # key metrics of one `ncu --set full` capture
    python tools/summarize_profiles.py full gpurun_out/bp.ncu-rep "header line" > profiles/rXX_ncu_bp.txt
"""
from __future__ import annotations

import csv
import io
import subprocess
import sys
from collections import defaultdict

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "launch__grid_size",
    "launch__block_size",
    "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic",
    "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed.avg.per_cycle_active",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__inst_executed.sum",
]


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10 and r[0] != "ID"]
    tot = defaultdict(float)
    cnt = defaultdict(int)
    for r in rows:
        if r[12] != "gpu__time_duration.sum":
            continue
        name = r[4].split("(")[0][:60]
        v = float(r[14].replace(",", ""))
        if r[13] == "ms":
            v *= 1e3
        elif r[13] == "ns":
            v *= 1e-3
        tot[name] += v
        cnt[name] += 1
    s = sum(tot.values()) or 1.0
    print("# cold-cache serialized times: compare SHARES, not absolutes")
    print(f"{'kernel':60s} {'launches':>9s} {'total_us':>12s} {'share':>7s}")
    for k in sorted(tot, key=lambda k: -tot[k]):
        print(f"{k:60s} {cnt[k]:9d} {tot[k]:12.1f} {100 * tot[k] / s:6.1f}%")


def full(rep, header):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    print(f"# {header}")
    for r in rows[2:]:
        print(f"\n## {r[h.index('Kernel Name')]}")
        for k in KEYS:
            if k in h:
                i = h.index(k)
                print(f"{k:75s} {r[i]} {units[i]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
