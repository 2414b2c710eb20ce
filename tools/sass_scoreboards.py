#!/usr/bin/env python3
"""Scoreboard use in the fast kernel's row loop (static SASS): the write
barrier ptxas gave every global load, and which other instructions set or
wait on the same barrier (a false dependency on a DRAM load).
  sass_scoreboards.py LIB.so MANGLED_SUBSTRING"""
import re
import subprocess
import sys


def ctl(hi):
    c = hi >> 41
    return dict(stall=c & 15, wr=(c >> 5) & 7, rd=(c >> 8) & 7, wait=(c >> 11) & 63)


def main(lib, key):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout.splitlines()
    ins, on, i = [], False, 0
    while i < len(out):
        line = out[i]
        if "Function :" in line:
            if on and ins:
                break
            on = key in line
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);\s+/\* (0x[0-9a-f]+) \*/", line)
        if on and m and i + 1 < len(out):
            m2 = re.match(r"\s+/\* (0x[0-9a-f]+) \*/", out[i + 1])
            if m2:
                ins.append((int(m.group(1), 16), m.group(2).strip(), ctl(int(m2.group(1), 16))))
                i += 1
        i += 1
    loops = []
    for a, t, c in ins:
        m = re.search(r"(0x[0-9a-f]+)\s*$", t)
        if "BRA" in t and m and int(m.group(1), 16) < a:
            loops.append((int(m.group(1), 16), a))

    def n(l, op):
        return sum(op in t for a, t, c in ins if l[0] <= a <= l[1])
    lo, hi = min((l for l in loops if n(l, "ATOMS") >= 24 and n(l, "STG") >= 3), key=lambda l: l[1] - l[0])
    body = [x for x in ins if lo <= x[0] <= hi]
    ldg_sb = sorted({c["wr"] for a, t, c in body if "LDG" in t and c["wr"] != 7})
    print(f"{lib}: row loop {lo:#x}-{hi:#x}, {len(body)} instructions; LDG write barriers {ldg_sb}")
    for a, t, c in body:
        if "LDG" in t:
            print(f"  {a:#x} {t[:58]:58s} wr {c['wr']}")
    for sb in ldg_sb:
        sets = [(a, t) for a, t, c in body if "LDG" not in t and (c["wr"] == sb or c["rd"] == sb)]
        waits = [(a, t) for a, t, c in body if c["wait"] >> sb & 1]
        print(f"  SB{sb}: also set by {len(sets)} non-LDG instructions ({', '.join(sorted({t.split()[0] if not t.startswith('@') else t.split()[1] for a, t in sets}))}); waited on by {len(waits)}")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
