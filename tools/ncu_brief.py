#!/usr/bin/env python3
"""One-screen summary of an .ncu-rep (first kernel): time, instructions,
issue/pipe utilisation, L1/shared wavefronts and bank conflicts, DRAM bytes,
occupancy and the stall reasons per issued instruction.
  ncu_brief.py REP [REP ...]"""
import csv
import io
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__occupancy_limit_shared_mem",
    "launch__occupancy_limit_registers", "launch__shared_mem_per_block_dynamic", "launch__registers_per_thread",
    "launch__grid_size", "smsp__thread_inst_executed.sum",
]


def brief(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, r = rows[0], rows[1], rows[2]
    d = dict(zip(hdr, zip(units, r)))
    lines = [f"# {rep}"]
    for w in WANT:
        if w in d:
            lines.append(f"{w:72s} {d[w][0]:10s} {d[w][1]}")
    for h in hdr:
        if "average_warps_issue_stalled" in h and h.endswith("per_issue_active.ratio"):
            v = float(d[h][1])
            if v > 0.02:
                lines.append(f"{h:72s} {'':10s} {v:.3f}")
    return "\n".join(lines)


if __name__ == "__main__":
    print("\n\n".join(brief(r) for r in sys.argv[1:]))
