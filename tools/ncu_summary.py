#!/usr/bin/env python3
"""Summarise an ncu --set full report (+ optional launch-list CSV) into a
markdown file under profiles/. Runs here (no GPU): ncu -i only."""
import csv
import subprocess
import sys


def details(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    kernel = rows[1][4] if len(rows) > 1 else "?"
    want = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "SM Frequency",
            "Executed Ipc Active", "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy",
            "Achieved Occupancy", "L1/TEX Hit Rate", "L2 Hit Rate", "Executed Instructions", "Grid Size",
            "Block Size", "Dynamic Shared Memory Per Block", "Warp Cycles Per Issued Instruction"]
    got = {}
    for r in rows:
        if len(r) > 14 and r[-4] in want and r[-4] not in got:
            got[r[-4]] = (r[-2], r[-3])
    return kernel, got


def raw(rep, keys):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, v = rows[0], rows[1], rows[2]  # header, units, values
    return {k: (v[h.index(k)] + " " + u[h.index(k)]).strip() for k in keys if k in h}


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    kn, mv, mn = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    tot = {}
    for r in rows[hi + 1:]:
        if len(r) > mv and r[mn] == "gpu__time_duration.sum":
            name = r[kn].split("(")[0]
            t, c = tot.get(name, (0.0, 0))
            tot[name] = (t + float(r[mv].replace(",", "")), c + 1)
    return tot


def main():
    rep, out = sys.argv[1], sys.argv[2]
    lcsv = sys.argv[3] if len(sys.argv) > 3 else None
    kernel, d = details(rep)
    rk = raw(rep, ["dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
                   "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
                   "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
                   "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
                   "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                   "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
                   "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
                   "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
                   "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio"])
    L = [f"# ncu summary: `{rep.split('/')[-1]}`", "", f"Kernel: `{kernel}`", "", "| metric | value |", "|---|---|"]
    for k, (val, unit) in d.items():
        L.append(f"| {k} | {val} {unit} |")
    for k, val in rk.items():
        L.append(f"| {k} | {val} |")
    if lcsv:
        tot = launches(lcsv)
        all_t = sum(t for t, _ in tot.values())
        L += ["", f"## Launch list (`{lcsv.split('/')[-1]}`, gpu__time_duration.sum, cold-cache, serialised)", "",
              "| kernel | launches | total ms | share |", "|---|---|---|---|"]
        for name, (t, c) in sorted(tot.items(), key=lambda x: -x[1][0]):
            L.append(f"| `{name}` | {c} | {t / 1e6:.3f} | {100 * t / all_t:.1f}% |")
    open(out, "w").write("\n".join(L) + "\n")
    print("\n".join(L))


if __name__ == "__main__":
    main()
