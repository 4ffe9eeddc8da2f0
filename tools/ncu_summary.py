#!/usr/bin/env python
"""Summarise ncu --set full reports (.ncu-rep) into a small JSON file for
profiles/: duration, DRAM traffic, pipe utilisation, occupancy and the top
stall reasons of each captured kernel.

  python tools/ncu_summary.py gpurun_out/prof_hair.ncu-rep > profiles/x.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.sum.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__inst_executed.sum", "smsp__sass_inst_executed_op_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__shared_mem_per_block_dynamic", "sm__cycles_elapsed.avg.per_second",
]
PFX, SFX = "smsp__average_warps_issue_stalled_", "_per_issue_active.ratio"


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    return r[0], r[1], r[2:]


def summarise(rep):
    head, units, data = rows(rep)
    res = []
    for v in data:
        d = {"report": rep.split("/")[-1], "kernel": v[head.index("Kernel Name")]}
        for k in KEYS:
            if k in head:
                d[k] = f"{v[head.index(k)]} {units[head.index(k)]}".strip()
        stalls = []
        for i, name in enumerate(head):
            if name.startswith(PFX) and name.endswith(SFX):
                try:
                    stalls.append((float(v[i]), name[len(PFX):-len(SFX)]))
                except ValueError:
                    pass
        d["stalls_per_issue_top"] = {n: round(x, 3) for x, n in sorted(stalls, reverse=True)[:8]}
        res.append(d)
    return res


def main():
    res = []
    for rep in sys.argv[1:]:
        res += summarise(rep)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
