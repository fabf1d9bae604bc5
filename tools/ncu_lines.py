"""Per-source-line instruction and stall-sample shares from an ncu report.

usage: python tools/ncu_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def lines(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source",
                          "cuda,sass"], capture_output=True, text=True).stdout
    cur, hdr, agg = None, None, {}
    for r in csv.reader(io.StringIO(raw)):
        if not r:
            continue
        if r[0] == "File Path":
            cur = r[1].split("/")[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or len(r) < 8 or r[2] != "-":
            continue
        try:
            ln = int(r[0])
        except ValueError:
            continue
        agg[(cur, ln)] = (int(r[7]), int(r[4]), r[1].strip()[:80])
    return agg


if __name__ == "__main__":
    agg = lines(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
    ti = sum(v[0] for v in agg.values()) or 1
    ts = sum(v[1] for v in agg.values()) or 1
    print(f"total instructions {ti}, stall samples {ts}")
    for (f, ln), (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{f:18s}{ln:5d} {100 * i / ti:5.1f}% inst {100 * s / ts:5.1f}% smpl  {src}")
