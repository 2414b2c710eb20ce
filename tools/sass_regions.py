#!/usr/bin/env python3
"""Per-region breakdown of an ncu source page (SASS view): executed
instructions and warp-stall samples of every backward-branch loop body and
of the straight-line code between them, largest first.
  ncu -i REP --page source --csv --print-source sass > src.csv
  sass_regions.py src.csv [N]"""
import csv
import re
import sys


def main(path, top=12):
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ia, isrc = hdr.index("Address"), hdr.index("Source")
    isamp, iexe = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    ins = []
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        ins.append((int(r[ia], 16), r[isrc].strip(), int(r[isamp] or 0), int(r[iexe] or 0)))
    base = ins[0][0]
    addr2i = {a: i for i, (a, *_) in enumerate(ins)}
    tot_s = sum(x[2] for x in ins)
    tot_e = sum(x[3] for x in ins)
    loops = []
    for i, (a, t, s, e) in enumerate(ins):
        m = re.search(r"BRA(?:\.\S+)?\s+(?:\S+,\s*)?(0x[0-9a-f]+)\s*$", t)
        if m:
            tgt = int(m.group(1), 16)
            tgt = tgt + base if tgt < base else tgt
            if tgt <= a and tgt in addr2i:
                loops.append((addr2i[tgt], i))
    # innermost loops first: attribute each instruction to the smallest loop containing it
    owner = [None] * len(ins)
    for s_, e_ in sorted(loops, key=lambda x: x[1] - x[0]):
        for k in range(s_, e_ + 1):
            if owner[k] is None:
                owner[k] = (s_, e_)
    agg = {}
    for k, (a, t, s, e) in enumerate(ins):
        key = owner[k] or ("straight",)
        d = agg.setdefault(key, [0, 0, 0])
        d[0] += s
        d[1] += e
        d[2] += 1
    print(f"total samples {tot_s}, warp-instructions executed {tot_e}")
    for key, (s, e, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        name = "straight-line code" if key == ("straight",) else \
            f"loop {hex(ins[key[0]][0] - base)}-{hex(ins[key[1]][0] - base)}"
        print(f"{name:32s} {n:5d} instr  samples {100 * s / tot_s:5.1f}%  executed {100 * e / tot_e:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 12)


def stall_mix(path, lo, hi):
    """Stall-reason mix of the instructions at offsets [lo, hi] (hex strings)."""
    rows = list(csv.reader(open(path)))
    hdr = rows[1]
    ia = hdr.index("Address")
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    base = int(rows[2][ia], 16)
    tot = dict.fromkeys(cols, 0)
    for r in rows[2:]:
        if len(r) < len(hdr):
            continue
        off = int(r[ia], 16) - base
        if int(lo, 16) <= off <= int(hi, 16):
            for c in cols:
                tot[c] += int(r[hdr.index(c)] or 0)
    s = sum(tot.values()) or 1
    return ", ".join(f"{c[6:]} {100 * v / s:.1f}%" for c, v in sorted(tot.items(), key=lambda kv: -kv[1]) if v)
