"""Novel-view rendering throughput on the C2 geometry.

Times, through the public API (host inputs, host outputs, wall clock around
each call after warm-up):
  * render_view(scene, view, channel)   -- rasterizer.py:206-215
  * render_scene_mask(scene, asn, view) -- maskrender.py:69-95, E objects
and, with --cpu, the oracle's render_view on a bounded sample of the same view
(one view, all host threads are not used: the oracle render is single-threaded).

usage: python tools/bench_render.py [--gaussians N] [--objects E] [--reps K] [--cpu]
"""

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2409_08270_b200 import Assignment, render_scene_mask, render_view, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gaussians", type=int, default=1_000_000)
    ap.add_argument("--objects", type=int, default=32)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--cpu", action="store_true")
    a = ap.parse_args()
    wl = synth.make_workload(seed=2, n_gaussians=a.gaussians, n_views=2, width=1008, height=756,
                             num_objects=a.objects)
    scene, view = wl.scene, wl.views[1]
    px = view.width * view.height
    ch = np.random.default_rng(0).random(len(scene))
    rng = np.random.default_rng(1)
    memb = np.zeros((a.objects, len(scene)), np.uint8)
    memb[rng.integers(0, a.objects, size=len(scene)), np.arange(len(scene))] = 1
    asn = Assignment(mode="scene", gamma=0.0, membership=memb)
    out = {}
    for name, fn in [("render_view", lambda: render_view(scene, view, ch)),
                     ("render_scene_mask", lambda: render_scene_mask(scene, asn, view))]:
        fn()
        t = []
        for _ in range(a.reps):
            t0 = time.perf_counter()
            fn()
            t.append(time.perf_counter() - t0)
        s = float(np.median(t))
        out[name] = {"s_per_view": s, "view_px_per_s": px / s}
    out["config"] = {"gaussians": len(scene), "image": f"{view.width}x{view.height}",
                     "objects": a.objects, "timing": "wall clock around the public call, "
                     "host inputs and outputs, median of reps"}
    if a.cpu:
        import oracle
        cam = oracle.camera_of(view)
        t0 = time.perf_counter()
        oracle.render_view(scene.means, scene.rotations, scene.scales, scene.opacities, cam, ch)
        s = time.perf_counter() - t0
        out["cpu_oracle_render_view"] = {"s_per_view": s, "view_px_per_s": px / s, "cores": 1}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
