#!/usr/bin/env python3
"""Opcode counts of the largest backward-branch loop body of one kernel in a
library (static SASS, no GPU): the row loop of the fast kernel.
  sass_loop.py LIB.so MANGLED_SUBSTRING"""
import collections
import re
import subprocess
import sys


def main(lib, key):
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    ins, on = [], False
    for line in out.splitlines():
        if "Function :" in line:
            on = key in line
            if on and ins:
                break
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
        if on and m:
            ins.append((int(m.group(1), 16), m.group(2).strip()))
    best = None
    for a, t in ins:
        m = re.search(r"BRA(?:\.\S+)?\s+(?:\S+,\s*)?`?\(?\.?L?_?x?_?(\w+)\)?\s*$", t)
        m2 = re.search(r"(0x[0-9a-f]+)\s*$", t)
        if "BRA" in t and m2:
            tgt = int(m2.group(1), 16)
            if tgt < a and (best is None or a - tgt > best[1] - best[0]):
                best = (tgt, a)
    # innermost loops only: the largest one is the 3-way unrolled row loop
    loops = []
    for a, t in ins:
        m2 = re.search(r"(0x[0-9a-f]+)\s*$", t)
        if "BRA" in t and m2 and int(m2.group(1), 16) < a:
            loops.append((int(m2.group(1), 16), a))
    inner = [l for l in loops if not any(o != l and l[0] <= o[0] and o[1] <= l[1] for o in loops)]
    for l in sorted(inner):
        b = [t for a, t in ins if l[0] <= a <= l[1]]
        print(f"  inner loop {l[0]:#x}-{l[1]:#x}: {len(b)} insts, ATOMS {sum('ATOMS' in t for t in b)}, LDG {sum('LDG' in t for t in b)}, STG {sum('STG' in t for t in b)}")
    if len(sys.argv) > 3:
        lo, hi = sorted(inner)[int(sys.argv[3])]
    else:
        # the 3-way unrolled row loop: the smallest loop with 24 shared atomics (8 pixels x 3 rows per lane)
        def n(l, op):
            return sum(op in t for a, t in ins if l[0] <= a <= l[1])
        lo, hi = min((l for l in loops if n(l, 'ATOMS') >= 24 and n(l, 'LDG') >= 3), key=lambda l: l[1] - l[0])
    body = [t for a, t in ins if lo <= a <= hi]
    c = collections.Counter(re.sub(r"^@!?U?P\d+\s+", "", t).split()[0].split(".")[0] for t in body)
    alu = {"VIMNMX", "VIMNMX3", "VIADDMNMX", "LOP3", "PRMT", "IADD3", "SHF", "SEL", "LEA", "ISETP", "IADD", "VIADD", "MOV"}
    print(f"{lib}: kernel insts {len(ins)}, loop body {len(body)}")
    for k, v in c.most_common():
        print(f"  {v:4d} {k}")
    print("  min/max ops", sum(v for k, v in c.items() if k.startswith("VI") and "MNMX" in k))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
