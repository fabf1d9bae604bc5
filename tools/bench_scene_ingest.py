"""End-to-end load_scene_ply -> solve on a C2-size checkpoint:
the reference-semantics host loader (numpy activations, float64 scene upload)
against the device path (raw float32 records uploaded, activated in K0).

usage: python tools/bench_scene_ingest.py [--gaussians 1000000] [--views 200] [--out JSON]
"""

import argparse
import json
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2409_08270_b200 import _native, export_ply, load_scene_ply, solve, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gaussians", type=int, default=1_000_000)
    ap.add_argument("--views", type=int, default=200)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    wl = synth.config_workload("C2", n_gaussians=a.gaussians, n_views=a.views)
    pairs = wl.pairs()
    with tempfile.TemporaryDirectory() as d:
        path = Path(d) / "scene.ply"
        export_ply(wl.scene, path)
        size = path.stat().st_size
        res = {}
        for name, dev in (("host_loader", None), ("device_loader", 0)):
            times, loads = [], []
            for r in range(a.reps + 1):
                ctx = _native.context(0)
                ctx._scene_key = None  # nothing resident: every rep uploads the scene
                t0 = time.perf_counter()
                sc = load_scene_ply(path, device=dev)
                t1 = time.perf_counter()
                M, asn = solve(sc, pairs, 2, 0.0, "binary")
                t2 = time.perf_counter()
                if r:  # first rep warms page cache, pools and workspaces
                    times.append(t2 - t0)
                    loads.append(t1 - t0)
                labels = asn.labels
            res[name] = {"s_load_plus_solve": float(np.median(times)),
                         "s_load": float(np.median(loads)), "fg": int(labels.sum())}
            res[name]["labels"] = labels
        same = bool(np.array_equal(res["host_loader"].pop("labels"),
                                   res["device_loader"].pop("labels")))
    out = {"workload": f"C2 scene ({a.gaussians} Gaussians) as a {size / 1e6:.0f} MB PLY, "
                       f"{a.views} views 1008x756, binary solve",
           "host_loader": res["host_loader"], "device_loader": res["device_loader"],
           "labels_identical": same,
           "scene_h2d_bytes": {"host_loader_float64": 88 * a.gaussians,
                               "device_loader_records": size}}
    print(json.dumps(out))
    if a.out:
        Path(a.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
