"""Repeated solves with changing scenes, object counts and paths (single context,
devices=[0, 0], LabelSolver re-assignment, render) -- device memory and host RSS
must plateau (grow-only scratch, pooled pinned blocks, cached contexts).

usage: python tools/stress_solve.py [--iters 60] [--out JSON]
"""

import argparse
import json
import resource
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2409_08270_b200 import LabelSolver, render_view, solve, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=60)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    wls = [synth.make_workload(seed=s, n_gaussians=n, n_views=6, width=320, height=240,
                               num_objects=e)
           for s, n, e in ((1, 200_000, 2), (2, 50_000, 9), (3, 120_000, 33))]
    trace = []
    for it in range(a.iters):
        wl = wls[it % len(wls)]
        e = wl.num_objects
        mode = "binary" if e == 2 else "scene"
        devices = [0, 0] if it % 2 else None
        M, asn = solve(wl.scene, wl.pairs(), e, 0.1, mode, devices=devices)
        s = LabelSolver(wl.scene)
        s.accumulate(wl.pairs(), e)
        s.assign(-0.2, mode)
        render_view(wl.scene, wl.views[0], np.ones(len(wl.scene)))
        free, total = torch.cuda.mem_get_info(0)
        rss = resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 1024
        trace.append({"iter": it, "device_used_mb": (total - free) / 2**20, "max_rss_mb": rss})
    first = trace[len(wls) * 2 - 1]
    last = trace[-1]
    out = {"iters": a.iters, "device_used_mb_after_warmup": first["device_used_mb"],
           "device_used_mb_end": last["device_used_mb"], "max_rss_mb_after_warmup": first["max_rss_mb"],
           "max_rss_mb_end": last["max_rss_mb"],
           "device_growth_mb": last["device_used_mb"] - first["device_used_mb"],
           "rss_growth_mb": last["max_rss_mb"] - first["max_rss_mb"]}
    print(json.dumps(out))
    if a.out:
        Path(a.out).write_text(json.dumps({"summary": out, "trace": trace}, indent=1))


if __name__ == "__main__":
    main()
