#!/usr/bin/env python3
"""Record the limiter counters of one ncu --set full capture of the fast
kernel in profiles/ncu_metrics.json, keyed by bench config, with the sha256 of
the library the capture ran (bench.py reports them next to its roofline and
says whether they belong to the library it loaded).

  ncu_to_json.py REP CONFIG PIXELS_PER_LAUNCH LIB [--out profiles/ncu_metrics.json]
"""
import argparse
import csv
import hashlib
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1810_11518_b200 import device_code_fingerprint  # noqa: E402


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, r = rows[0], rows[1], rows[2]
    return {h: (u, v) for h, u, v in zip(hdr, units, r)}


def num(d, key, unit_to=None):
    u, v = d[key]
    x = float(v.replace(",", ""))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
             "ms": 1e-3, "msecond": 1e-3, "s": 1.0}
    if unit_to == "B":
        return x * scale[u]
    if unit_to == "s":
        return x * scale[u]
    return x


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("config")
    ap.add_argument("pixels", type=float)
    ap.add_argument("lib")
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "ncu_metrics.json"))
    a = ap.parse_args()
    d = raw(a.rep)
    px = a.pixels
    t = num(d, "gpu__time_duration.sum", "s")
    rd = num(d, "dram__bytes_read.sum", "B")
    wr = num(d, "dram__bytes_write.sum", "B")
    inst = num(d, "smsp__inst_executed.sum")
    rec = {
        "kernel_time_s_cold": t,
        "dram_read_bytes_per_px": round(rd / px, 4),
        "dram_write_bytes_per_px": round(wr / px, 4),
        "dram_bytes_per_px": round((rd + wr) / px, 4),
        "thread_inst_per_px": round(inst * 32 / px, 2),
        "issue_active_pct": round(num(d, "smsp__issue_active.avg.pct_of_peak_sustained_active"), 1),
        "alu_pipe_pct": round(num(d, "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active"), 1),
        "fma_pipe_pct": round(num(d, "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"), 1),
        "l1_data_pipe_pct": round(num(d, "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"), 1),
        "dram_throughput_pct": round(num(d, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), 1),
        "shared_bank_conflicts_per_px": round(num(d, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum") / px, 3),
        "warps_active_pct": round(num(d, "sm__warps_active.avg.pct_of_peak_sustained_active"), 1),
        "pixels_per_launch": px,
        "source": os.path.relpath(os.path.abspath(a.rep), ROOT),
        "lib_sha256": hashlib.sha256(open(a.lib, "rb").read()).hexdigest(),
        "device_code_sha256": device_code_fingerprint(a.lib),
    }
    db = {}
    if os.path.exists(a.out):
        db = json.load(open(a.out))
    db[a.config] = rec
    with open(a.out, "w") as f:
        json.dump(db, f, indent=1, sort_keys=True)
    print(json.dumps({a.config: rec}, indent=1))


if __name__ == "__main__":
    main()
