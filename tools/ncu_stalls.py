"""Stall reasons per issued instruction + eligible/active warps from an ncu report.

usage: python tools/ncu_stalls.py REPORT.ncu-rep > profiles/r1_raster_stalls_c2.json
"""
import csv
import io
import json
import subprocess
import sys

PFX = "smsp__average_warps_issue_stalled_"
SFX = "_per_issue_active.ratio"


def stalls(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, vals = rows[0], rows[2]
    out = {}
    for k, v in zip(head, vals):
        if k.startswith(PFX) and k.endswith(SFX) and "not_issued" not in k:
            try:
                x = float(v)
            except ValueError:
                continue
            if x > 0.05:
                out[k[len(PFX):-len(SFX)]] = x
    get = dict(zip(head, vals))
    return {
        "kernel": get.get("Kernel Name", "")[:80],
        "stall_cycles_per_issued_instruction": dict(sorted(out.items(), key=lambda t: -t[1])),
        "warps_eligible_per_cycle": float(get["smsp__warps_eligible.avg.per_cycle_active"]),
        "warps_active_per_scheduler": float(get["smsp__warps_active.avg.per_cycle_active"]),
        "issue_active_pct": float(get["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
    }


if __name__ == "__main__":
    print(json.dumps(stalls(sys.argv[1]), indent=1))
