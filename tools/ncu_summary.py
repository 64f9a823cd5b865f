#!/usr/bin/env python
"""Summarise an ncu --set full report (read here, no GPU): key throughput, traffic, occupancy
and stall metrics per profiled kernel, as JSON.

    python tools/ncu_summary.py gpurun_out/prof_r1a.ncu-rep [--algo-bytes N]
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "lts__t_bytes.sum", "lts__t_sectors_op_read.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "launch__shared_mem_per_block_static", "launch__grid_size", "launch__block_size",
    "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_selected_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_drain_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_membar_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_imc_miss_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_tex_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio",
    "smsp__cycles_active.avg", "sm__cycles_elapsed.avg", "gpc__cycles_elapsed.max",
]


SCALE = {"byte": (1, "byte"), "Kbyte": (1e3, "byte"), "Mbyte": (1e6, "byte"),
         "Gbyte": (1e9, "byte"), "ns": (1, "ns"), "us": (1e3, "ns"), "usecond": (1e3, "ns"),
         "ms": (1e6, "ns"), "msecond": (1e6, "ns"), "nsecond": (1, "ns")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--algo-bytes", type=float, default=None)
    args = ap.parse_args()
    out = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        d = {"kernel": row[hdr.index("Kernel Name")][:80]}
        for m in METRICS:
            if m in hdr:
                v = row[hdr.index(m)]
                u = units[hdr.index(m)]
                try:
                    d[m] = float(v.replace(",", ""))
                    if u in SCALE:  # normalise bytes to byte and time to ns
                        d[m] *= SCALE[u][0]
                        u = SCALE[u][1]
                except ValueError:
                    d[m] = v
                if u:
                    d[m + " [unit]"] = u
        if args.algo_bytes and "dram__bytes_read.sum" in d:
            dram = d["dram__bytes_read.sum"] + d.get("dram__bytes_write.sum", 0)
            d["dram_over_algorithmic"] = dram / args.algo_bytes
        res.append(d)
    json.dump(res, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
