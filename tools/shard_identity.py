"""Determinism at full benchmark size: one GPU solve vs the
same scene split over 8 contexts (devices=[0]*8: the single-process multi-GPU
path -- dynamic view queue, 8 accumulators reduced slice by slice in the
finalize), and vs a second single-GPU solve, with the fixed-point accumulator
(default) and with float64 atomics.

usage: python tools/shard_identity.py [--configs C2,C3,C4] [--out JSON]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2409_08270_b200 import solve, synth  # noqa: E402


def compare(a, b):
    return {"matrix_bit_identical": bool(np.array_equal(a[0], b[0])),
            "entries_differing": int(np.count_nonzero(a[0] != b[0])),
            "max_abs_diff": float(np.abs(a[0] - b[0]).max()),
            "label_flips": int(np.count_nonzero(a[1] != b[1]))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3,C4")
    ap.add_argument("--shards", type=int, default=8)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    res = {}
    for cfg in a.configs.split(","):
        t0 = time.perf_counter()
        wl = synth.config_workload(cfg)
        pairs = wl.pairs()
        e = wl.num_objects
        mode = "binary" if e == 2 else "scene"
        rec = {"views": len(wl.views), "gaussians": len(wl.scene), "E": e,
               "gen_s": time.perf_counter() - t0}
        for det in (True, False):
            def run(devices=None):
                st = {}
                M, asn = solve(wl.scene, pairs, e, 0.0, mode, devices=devices,
                               deterministic=det, stats=st)
                lab = asn.labels if mode == "binary" else asn.membership
                return np.array(M.values), np.array(lab), st
            one = run()
            again = run()
            multi = run([0] * a.shards)
            key = "fixed" if det else "f64"
            rec[key] = {"rerun": compare(one, again),
                        f"{a.shards}_contexts": compare(one, multi),
                        "views_per_context": multi[2].get("views_per_device")}
        res[cfg] = rec
        print(cfg, json.dumps(rec), flush=True)
        del wl, pairs
    if a.out:
        Path(a.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
