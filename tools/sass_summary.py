"""Per-kernel SASS summary of the product library (cuobjdump -sass): instruction
count and the opcodes that prove the design choices -- UBLKCP / SYNCS (TMA bulk
copies + mbarriers), REDG (fixed-point / float64 accumulator REDs), MATCH, SHFL,
MUFU, float64 arithmetic, global / shared memory traffic.

usage: python tools/sass_summary.py [LIB] > profiles/r2_sass_summary.json
"""
import json
import re
import subprocess
import sys
from collections import Counter

LIB = sys.argv[1] if len(sys.argv) > 1 else "paper_2409_08270_b200/_lib/libflashsplat_b200.so"
KEEP = re.compile(r"^(UBLKCP|SYNCS|REDG|RED|ATOM|MATCH|SHFL|MUFU|DADD|DMUL|DFMA|LDG|STG|LDS|STS|"
                  r"BAR|REDUX|VOTE|ATOMS|I2F\.F64|F2I\.F64|HADD2|F2FP)")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True,
                          check=True).stdout
    out, name, ops, count = {}, None, Counter(), 0
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            if name:
                out[name] = {"instructions": count, "selected": dict(sorted(ops.items()))}
            name, ops, count = m.group(1), Counter(), 0
            continue
        m = re.match(r"\s+/\*[0-9a-f]{4,}\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", line)
        if name and m:
            count += 1
            if KEEP.match(m.group(1)):
                ops[m.group(1)] += 1
    if name:
        out[name] = {"instructions": count, "selected": dict(sorted(ops.items()))}
    json.dump(out, sys.stdout, indent=1)


if __name__ == "__main__":
    main()
