"""Interactive gamma re-assignment on a device-resident matrix (
reference service.py:56-66,101-127, test_service.py:162-179 asks < 200 ms).

Builds a synthetic E x N float32 matrix on the device once, then times
LabelSolver.assign(gamma) -- one argmax launch plus the labels' D2H into
pinned memory -- and the reference-equivalent host member counts.

usage: python tools/bench_assign.py [--gaussians N] [--objects E] [--reps K]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2409_08270_b200 import GaussianScene  # noqa: E402
from paper_2409_08270_b200.solve import LabelSolver  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gaussians", type=int, default=1_000_000)
    ap.add_argument("--objects", type=int, nargs="+", default=[2, 32])
    ap.add_argument("--reps", type=int, default=20)
    a = ap.parse_args()
    n = a.gaussians
    rng = np.random.default_rng(0)
    scene = GaussianScene(rng.random((n, 3)), np.tile([1.0, 0, 0, 0], (n, 1)),
                          np.full((n, 3), 0.01), np.full(n, 0.5))
    out = {}
    for e in a.objects:
        s = LabelSolver(scene)
        A = s.ctx.alloc(4 * e * n)
        A.from_host(rng.random((e, n), dtype=np.float32))
        s._A_cur, s._out_cur = A, s.ctx.alloc(e * n)
        s.num_objects = e
        mode = "binary" if e == 2 else "scene"
        counts0 = s.assign(0.0, mode).member_counts()
        t = []
        for i in range(a.reps):
            g = -1.0 + 2.0 * i / max(a.reps - 1, 1)
            t0 = time.perf_counter()
            asn = s.assign(g, mode)
            counts = asn.member_counts()
            t.append(time.perf_counter() - t0)
        out[f"E{e}"] = {"ms_per_assign": 1e3 * float(np.median(t)), "gaussians": n,
                        "mode": mode, "member_counts_gamma0": counts0[:4]}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
