#!/usr/bin/env python3
"""Summarise ncu reports into the markdown/JSON kept under profiles/.

usage: ncu_summary.py OUT_PREFIX REPORT.ncu-rep|REPORT.raw.csv [...]
Reads each report with `ncu -i --page raw --csv` (no GPU needed) and writes
OUT_PREFIX.md (table of the counters the north star asks for) and
OUT_PREFIX.json (the same values, machine readable).
"""
import csv
import io
import json
import os
import subprocess
import sys

METRICS = [
    ("duration", "gpu__time_duration.sum"),
    ("SM clock", "sm__cycles_elapsed.avg.per_second"),
    ("grid x block", None),
    ("registers/thread", "launch__registers_per_thread"),
    ("warps active (% of peak)", "sm__warps_active.avg.pct_of_peak_sustained_active"),
    ("FP64 pipe active (%)", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
    ("issue slots busy (%)", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
    ("DFMA lanes/cycle/SMSP", "smsp__sass_thread_inst_executed_op_dfma_pred_on.avg.per_cycle_elapsed"),
    ("DMUL lanes/cycle/SMSP", "smsp__sass_thread_inst_executed_op_dmul_pred_on.avg.per_cycle_elapsed"),
    ("DADD lanes/cycle/SMSP", "smsp__sass_thread_inst_executed_op_dadd_pred_on.avg.per_cycle_elapsed"),
    ("smem load wavefronts", "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum"),
    ("smem load bank conflicts", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum"),
    ("L1TEX throughput (%)", "l1tex__throughput.avg.pct_of_peak_sustained_active"),
    ("L1 hit rate (%)", "l1tex__t_sector_hit_rate.pct"),
    ("L2 hit rate (%)", "lts__t_sector_hit_rate.pct"),
    ("DRAM read", "dram__bytes_read.sum"),
    ("DRAM write", "dram__bytes_write.sum"),
    ("DRAM write rate", "dram__bytes_write.sum.per_second"),
    ("stall: math pipe throttle", "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio"),
    ("stall: not selected", "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio"),
    ("stall: wait", "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"),
    ("stall: long scoreboard", "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio"),
    ("stall: short scoreboard", "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio"),
    ("stall: dispatch", "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio"),
]


def raw(rep):
    # a report, or its `ncu -i REPORT --page raw --csv` export (made on the GPU
    # box when the report itself is too large to bring back)
    if rep.endswith(".csv"):
        out = open(rep).read()
    else:
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                             text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return {h: (v, u) for h, u, v in zip(rows[0], rows[1], rows[2])}


def main():
    prefix, reps = sys.argv[1], sys.argv[2:]
    data = {}
    for rep in reps:
        d = raw(rep)
        name = os.path.basename(rep).replace(".ncu-rep", "").replace(".raw.csv", "")
        vals = {"kernel": d.get("Kernel Name", ("?", ""))[0]}
        for label, key in METRICS:
            if key is None:
                vals[label] = f"{d.get('launch__grid_size', ('?',))[0]} x " \
                              f"{d.get('launch__block_size', ('?',))[0]}"
            elif key in d:
                vals[label] = f"{d[key][0]} {d[key][1]}".strip()
        data[name] = vals
    json.dump(data, open(prefix + ".json", "w"), indent=1)
    names = list(data)
    with open(prefix + ".md", "w") as f:
        f.write("| metric | " + " | ".join(names) + " |\n")
        f.write("|---|" + "---|" * len(names) + "\n")
        f.write("| kernel | " + " | ".join(data[n]["kernel"][:60] for n in names) + " |\n")
        for label, _ in METRICS:
            f.write(f"| {label} | " + " | ".join(data[n].get(label, "") for n in names) + " |\n")
    print(open(prefix + ".md").read())


if __name__ == "__main__":
    main()
